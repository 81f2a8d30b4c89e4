// C ABI of libsplatcull_b200.so: argument checks, workspace carving and the
// per-frame stage orchestration.  See include/splatcull_b200.h.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "common.cuh"

namespace sc {
cudaError_t launch_count_used(const float *cmax, const unsigned long long *n_dev, int64_t n_max,
                              sc_frame_stats *stats, cudaStream_t st);
cudaError_t launch_labels_or(const float *cmax, int64_t n, uint32_t *bits, cudaStream_t st);
}

namespace sc {
int sm_count()
{
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const bool cached = dev >= 0 && dev < 64;
    int n = cached ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (n > 0) return n;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
    if (cached) cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

cudaError_t smem_attr_once(const void *func, int bytes)
{
    static std::mutex mu;
    static std::unordered_map<const void *, unsigned long long> done;   // func -> bitmask of devices
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = (dev >= 0 && dev < 64) ? 1ull << dev : 0ull;
    {
        std::lock_guard<std::mutex> g(mu);
        if (bit && (done[func] & bit)) return cudaSuccess;
    }
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit) {
        std::lock_guard<std::mutex> g(mu);
        done[func] |= bit;
    }
    return e;
}
}  // namespace sc

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

extern "C" void sc_note_launch(void) { g_launches.fetch_add(1, std::memory_order_relaxed); }

static int fail(int code, const char *fmt, const char *detail = "")
{
    char buf[512];
    snprintf(buf, sizeof(buf), fmt, detail);
    g_last_error = buf;
    return code;
}

static int cuda_status(cudaError_t e, const char *where)
{
    if (e == cudaSuccess) return SC_OK;
    char buf[512];
    snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
    g_last_error = buf;
    return SC_ERR_CUDA;
}

#define SC_TRY(expr, where)                                  \
    do {                                                     \
        int _rc = cuda_status((expr), where);                \
        if (_rc != SC_OK) return _rc;                        \
    } while (0)

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

struct Layout {
    size_t inst, chunk_state, chunk_cnt, chunk_inst, chunk_stage, ctr, surv, splats, wins, key_a, key_b, pv_a, pv_b, depth64, rect, ekey_a, ekey_b,
        eval_a, eval_b, tile_off, task_order, boff, rs_counts, scan_part, total;
    int64_t max_chunks, nblk_max, n_tiles, n_tiles_ref;
    int n_tx, n_ty, n_tx_ref;
};

constexpr int kMaxTileSize = 65535;

// Workspace layout.  Two regions are unions of buffers with disjoint lifetimes
// (stream order within one frame):
//   U = [surv | key_a | key_b | pv_b]          cull -> projection -> depth sort -> tie-fix
//     = [ekey_b | eval_b]                      block / entry sort ping-pong (after the emission)
//   V = [chunk_stage]                          cull staging
//     = [depth64 | rect]                       stage API: projection -> tie-fix / entry counts
//     = [ekey_a | eval_a]                      emission -> block sort -> blend
// key_b doubles as the projection's deferred-splat list, the tie-run list and the
// emission's per-warp totals; pv_b (the depth sort's other payload) holds the
// f64 depths of long tie runs.  Per survivor: splats 32 + wins 8 + pv_a 8 + U 24 B.
Layout layout(int64_t n_inst, int64_t max_pairs, int64_t capS, int64_t capE, int32_t w, int32_t h, int32_t ts)
{
    Layout L{};
    L.n_tx = (w + sc::kTile - 1) / sc::kTile;
    L.n_ty = (h + sc::kTile - 1) / sc::kTile;
    L.n_tiles = (int64_t)L.n_tx * L.n_ty;
    L.n_tx_ref = (w + ts - 1) / ts;
    L.n_tiles_ref = (int64_t)L.n_tx_ref * ((h + ts - 1) / ts);
    L.max_chunks = max_pairs / sc::kChunk + n_inst + 1;
    const int64_t big = std::max<int64_t>(std::max<int64_t>(capS, capE), 1);
    L.nblk_max = (big + sc::kRadixTile - 1) / sc::kRadixTile;
    const int64_t part = (std::max<int64_t>(256 * L.nblk_max, big) + sc::kScanTile - 1) / sc::kScanTile + 1;
    // key buffers also hold small per-tile lists: at least 4096 words
    const int64_t capK = std::max<int64_t>(capS, 4096);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + std::max<size_t>(bytes, 1));
        return o;
    };
    L.inst = take(sizeof(sc::InstFrame) * (size_t)std::max<int64_t>(n_inst, 1));
    L.chunk_state = take(sizeof(unsigned long long) * (size_t)L.max_chunks);
    L.chunk_cnt = take(sizeof(uint32_t) * (size_t)L.max_chunks);
    L.chunk_inst = take(sizeof(uint32_t) * (size_t)L.max_chunks);
    L.ctr = take(sizeof(sc::Counters));
    L.splats = take(sizeof(sc_splat) * (size_t)capS);
    L.wins = take(sizeof(sc_window) * (size_t)capS);
    // +16 bytes: radix bulk copies round the last tile up to 16 bytes
    L.pv_a = take(8 * (size_t)capS + 16);
    // region U
    {
        const size_t u0 = off;
        size_t o = 0;
        auto sub = [&](size_t bytes) { size_t r = o; o = align_up(o + std::max<size_t>(bytes, 1)); return u0 + r; };
        L.surv = sub(sizeof(sc_survivor) * (size_t)capS);
        L.key_a = sub(4 * (size_t)capK + 16);
        L.key_b = sub(4 * (size_t)capK + 16);
        L.pv_b = sub(8 * (size_t)capS + 16);
        const size_t u_a = o;
        o = 0;
        L.ekey_b = sub(4 * (size_t)capE + 16);
        L.eval_b = sub(4 * (size_t)capE + 16);
        off = align_up(u0 + std::max(u_a, o));
    }
    // region V
    {
        const size_t v0 = off;
        size_t o = 0;
        auto sub = [&](size_t bytes) { size_t r = o; o = align_up(o + std::max<size_t>(bytes, 1)); return v0 + r; };
        L.chunk_stage = sub(sizeof(uint16_t) * (size_t)L.max_chunks * sc::kChunk);
        const size_t v_a = o;
        o = 0;
        L.depth64 = sub(8 * (size_t)capS);
        L.rect = sub(8 * (size_t)capS);
        const size_t v_b = o;
        o = 0;
        L.ekey_a = sub(4 * (size_t)capE + 16);
        L.eval_a = sub(4 * (size_t)capE + 16);
        off = align_up(v0 + std::max(std::max(v_a, v_b), o));
    }
    L.tile_off = take(4 * (size_t)(L.n_tiles_ref + 1));
    L.task_order = take(4 * (size_t)(8 * L.n_tiles));   // blend dispatch order over (tile, block) lists
    L.boff = take(4 * (size_t)(8 * L.n_tiles + 1));
    L.rs_counts = take(4 * (size_t)(256 * L.nblk_max));
    L.scan_part = take(4 * (size_t)part);
    L.total = off;
    return L;
}

int carve(const sc_workspace *ws, int32_t w, int32_t h, int32_t ts, sc::Ws &out)
{
    if (!ws || !ws->base) return fail(SC_ERR_INVALID, "workspace is NULL%s");
    if (ws->cap_survivors < 0 || ws->cap_entries < 0 || ws->cap_survivors > 0xFFFFFFF0ll ||
        ws->cap_entries > 0xFFFFFFF0ll || ws->n_instances < 0 || ws->max_pairs < 0)
        return fail(SC_ERR_INVALID, "workspace capacities out of range%s");
    Layout L = layout(ws->n_instances, ws->max_pairs, ws->cap_survivors, ws->cap_entries, w, h, ts);
    if (ws->bytes < L.total) return fail(SC_ERR_INVALID, "workspace too small for these capacities and tile size%s");
    char *b = static_cast<char *>(ws->base);
    out.inst = reinterpret_cast<sc::InstFrame *>(b + L.inst);
    out.chunk_state = reinterpret_cast<unsigned long long *>(b + L.chunk_state);
    out.chunk_cnt = reinterpret_cast<uint32_t *>(b + L.chunk_cnt);
    out.chunk_inst = reinterpret_cast<uint32_t *>(b + L.chunk_inst);
    out.chunk_stage = reinterpret_cast<uint16_t *>(b + L.chunk_stage);
    out.ctr = reinterpret_cast<sc::Counters *>(b + L.ctr);
    out.surv = reinterpret_cast<sc_survivor *>(b + L.surv);
    out.splats = reinterpret_cast<sc_splat *>(b + L.splats);
    out.wins = reinterpret_cast<sc_window *>(b + L.wins);
    out.key_a = reinterpret_cast<uint32_t *>(b + L.key_a);
    out.key_b = reinterpret_cast<uint32_t *>(b + L.key_b);
    out.pv_a = reinterpret_cast<uint2 *>(b + L.pv_a);
    out.pv_b = reinterpret_cast<uint2 *>(b + L.pv_b);
    out.depth64 = reinterpret_cast<double *>(b + L.depth64);
    out.rect = reinterpret_cast<ushort4 *>(b + L.rect);
    out.ekey_a = reinterpret_cast<uint32_t *>(b + L.ekey_a);
    out.ekey_b = reinterpret_cast<uint32_t *>(b + L.ekey_b);
    out.eval_a = reinterpret_cast<uint32_t *>(b + L.eval_a);
    out.eval_b = reinterpret_cast<uint32_t *>(b + L.eval_b);
    out.tile_off = reinterpret_cast<uint32_t *>(b + L.tile_off);
    out.task_order = reinterpret_cast<uint32_t *>(b + L.task_order);
    out.boff = reinterpret_cast<uint32_t *>(b + L.boff);
    out.rs_counts = reinterpret_cast<uint32_t *>(b + L.rs_counts);
    out.scan_part = reinterpret_cast<uint32_t *>(b + L.scan_part);
    out.capS = ws->cap_survivors;
    out.capE = ws->cap_entries;
    out.max_chunks = L.max_chunks;
    out.nblk_max = L.nblk_max;
    out.n_tiles = L.n_tiles;
    out.n_tx = L.n_tx;
    out.n_ty = L.n_ty;
    out.ts = ts;
    out.n_tx_ref = L.n_tx_ref;
    out.n_tiles_ref = L.n_tiles_ref;
    return SC_OK;
}

int check_camera(const sc_camera *cam)
{
    if (!cam) return fail(SC_ERR_INVALID, "camera is NULL%s");
    if (cam->width <= 0 || cam->height <= 0 || cam->width > 32000 || cam->height > 32000)
        return fail(SC_ERR_INVALID, "camera size out of range%s");
    // frame-path block sort key: (8 x 16x16-tile id + block) << 10 must fit 32 bits
    const int64_t n_tiles16 = (int64_t)((cam->width + sc::kTile - 1) / sc::kTile) * ((cam->height + sc::kTile - 1) / sc::kTile);
    if (8 * n_tiles16 >= (1ll << 22)) return fail(SC_ERR_INVALID, "camera has too many pixels (> ~134 Mpx)%s");
    if (!(cam->focal > 0.0)) return fail(SC_ERR_INVALID, "camera focal must be positive%s");
    return SC_OK;
}

int check_opts(const sc_opts *o)
{
    if (!o) return fail(SC_ERR_INVALID, "opts is NULL%s");
    if (o->tile_size < 1 || o->tile_size > kMaxTileSize) return fail(SC_ERR_INVALID, "tile_size must be in [1, 65535]%s");
    if (o->frustum_mode < SC_FRUSTUM_MARGIN || o->frustum_mode > SC_FRUSTUM_OFF)
        return fail(SC_ERR_INVALID, "unknown frustum_mode%s");
    if (o->band_y1 > 0) {
        if (o->tile_size != sc::kTile) return fail(SC_ERR_UNSUPPORTED, "screen bands need tile_size 16%s");
        if (o->band_y0 < 0 || o->band_y0 % sc::kTile != 0 || o->band_y1 <= o->band_y0)
            return fail(SC_ERR_INVALID, "band must be [y0, y1) with y0 a multiple of 16 and y1 > y0%s");
    }
    return SC_OK;
}

int check_scene(const sc_scene *s)
{
    if (!s) return fail(SC_ERR_INVALID, "scene is NULL%s");
    if (s->n_instances < 0 || s->n_gauss < 0 || s->n_assets < 0 || s->n_pairs < 0)
        return fail(SC_ERR_INVALID, "negative scene sizes%s");
    if (s->n_instances > 0 && (!s->instances || !s->assets))
        return fail(SC_ERR_INVALID, "scene tables are NULL%s");
    if (s->n_gauss > 0 && (!s->mean_opa || !s->quat || !s->scale_smax || !s->sh || !s->appear))
        return fail(SC_ERR_INVALID, "scene gaussian arrays are NULL%s");
    if (s->sh_stride < 3) return fail(SC_ERR_INVALID, "sh_stride must be >= 3%s");
    return SC_OK;
}

// the cull writes per-instance and per-chunk state sized by the workspace: the scene
// must fit it (k_prep also refuses, on the device, chunk totals beyond max_chunks)
int check_fit(const sc_scene *s, const sc_workspace *ws)
{
    if (ws && (ws->n_instances < s->n_instances || ws->max_pairs < s->n_pairs))
        return fail(SC_ERR_INVALID, "workspace was sized for a smaller scene (n_instances / max_pairs)%s");
    return SC_OK;
}

}  // namespace

namespace sc {
__global__ void k_set_survivors(Counters *ctr, sc_frame_stats *stats, int64_t n)
{
    ctr->survivors = (unsigned long long)n;
    stats->survivors = n;
}

// dst[i] = src[i] for i < min(*n_dev, cap) (words; copy-outs of device-counted lists)
__global__ void k_copy_words(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst,
                             const unsigned long long *n_dev, int64_t cap, int words_per_item)
{
    const int64_t n = std::min<int64_t>((int64_t)*n_dev, cap) * words_per_item;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t copy_counted(const void *src, void *dst, const unsigned long long *n_dev, int64_t cap, int words,
                         cudaStream_t st)
{
    if (cap <= 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((cap * words + 255) / 256, (int64_t)sm_count() * 8));
    SC_LAUNCH(k_copy_words, grid, 256, 0, st, static_cast<const uint32_t *>(src), static_cast<uint32_t *>(dst), n_dev,
              cap, words);
    return cudaGetLastError();
}
}  // namespace sc

namespace {
// Stages (c)-(e) of the frame path over w.surv (count in ctr->survivors), plus
// the optional debug copies.  mark(i) records the caller's stage events.
template <typename Mark>
int frame_tail(const sc_scene *scene, const sc_camera *cam, const sc_opts *opts, const sc::Ws &w,
               const sc_frame_out *out, cudaStream_t st, Mark &&mark)
{
    sc_frame_stats *stats = out->stats;
    const sc_frame_debug *dbg = out->debug;
    // the survivor list shares region U with the block sort: copy it out now
    if (out->survivors)
        SC_TRY(sc::copy_counted(w.surv, out->survivors, &w.ctr->survivors, w.capS, 2, st), "copy survivors");
    SC_TRY(sc::launch_project(*scene, w.surv, &w.ctr->survivors, w.capS, *cam, *opts, w.splats, w.wins, nullptr,
                              nullptr, w.key_a, w.pv_a, nullptr, nullptr, nullptr, stats, w.ctr, w.key_b, st),
           "project");
    SC_TRY(mark(2), "event");
    uint32_t *order = nullptr, *entries = nullptr;
    uint32_t *bkeys = nullptr;
    SC_TRY(sc::launch_bin(w, *scene, w.surv, &w.ctr->survivors, w.capS, *cam, w.wins, stats, true, &order, &entries,
                          &bkeys, dbg ? dbg->order : nullptr, st),
           "bin/sort");
    SC_TRY(mark(3), "event");
    if (dbg) {
        if (dbg->block_offsets)
            SC_TRY(cudaMemcpyAsync(dbg->block_offsets, w.boff, 4 * (size_t)(8 * w.n_tiles + 1), cudaMemcpyDeviceToDevice,
                                   st), "copy block offsets");
        if (dbg->block_entries)
            SC_TRY(sc::copy_counted(entries, dbg->block_entries, &w.ctr->entries_eff, w.capE, 1, st), "copy block entries");
        if (dbg->block_codes)
            SC_TRY(sc::copy_counted(bkeys, dbg->block_codes, &w.ctr->entries_eff, w.capE, 1, st), "copy block codes");
    }
    if (opts->record_contributions && w.capS > 0)
        SC_TRY(cudaMemsetAsync(out->contrib_max, 0, 4 * (size_t)w.capS, st), "memset contrib_max");
    const sc::BlendLists lists{w.boff, entries, bkeys, nullptr, true, w.ctr};
    SC_TRY(sc::launch_blend(w.splats, lists, *cam, *opts, *out, w.capS, w.task_order, st), "blend");
    SC_TRY(mark(4), "event");
    if (opts->record_contributions)
        SC_TRY(sc::launch_count_used(out->contrib_max, &w.ctr->survivors, w.capS, stats, st), "count used");
    return SC_OK;
}

int check_frame_out(const sc_frame_out *out, const sc_opts *opts)
{
    if (!out || !out->image || !out->trans || !out->stats) return fail(SC_ERR_INVALID, "output buffers are NULL%s");
    if (opts->record_contributions && (!out->contrib_max || !out->contrib_sum))
        return fail(SC_ERR_INVALID, "record_contributions needs contrib_max and contrib_sum%s");
    return SC_OK;
}

}  // namespace

extern "C" {

int sc_abi_version(void) { return SC_ABI_VERSION; }
const char *sc_last_error(void) { return g_last_error.c_str(); }
int64_t sc_kernel_launches(void) { return (int64_t)g_launches.load(); }

size_t sc_workspace_bytes(int64_t n_instances, int64_t max_pairs, int64_t cap_survivors, int64_t cap_entries,
                          int32_t width, int32_t height, int32_t tile_size)
{
    if (tile_size < 1 || tile_size > kMaxTileSize || width <= 0 || height <= 0 || cap_survivors < 0 ||
        cap_entries < 0 || n_instances < 0 || max_pairs < 0)
        return 0;
    return layout(n_instances, max_pairs, cap_survivors, cap_entries, width, height, tile_size).total;
}

int sc_cull_mlp(const sc_scene *scene, const sc_camera *cam, const sc_opts *opts, const sc_workspace *ws,
                sc_survivor *survivors, int64_t cap_survivors, sc_frame_stats *stats, void *stream)
{
    int rc;
    if ((rc = check_scene(scene)) || (rc = check_camera(cam)) || (rc = check_opts(opts))) return rc;
    if (!stats) return fail(SC_ERR_INVALID, "stats is NULL%s");
    if (survivors && cap_survivors < 0) return fail(SC_ERR_INVALID, "cap_survivors must be >= 0%s");
    sc::Ws w;
    if ((rc = carve(ws, cam->width, cam->height, opts->tile_size, w)) || (rc = check_fit(scene, ws))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SC_TRY(cudaMemsetAsync(stats, 0, sizeof(sc_frame_stats), st), "memset stats");
    SC_TRY(cudaMemsetAsync(w.ctr, 0, sizeof(sc::Counters), st), "memset counters");
    SC_TRY(sc::launch_prep(*scene, *cam, *opts, w, stats, st), "prep");
    SC_TRY(sc::launch_cull(*scene, *cam, *opts, w, survivors ? survivors : w.surv,
                           survivors ? cap_survivors : w.capS, stats, st),
           "cull");
    return SC_OK;
}

int sc_project(const sc_scene *scene, const sc_survivor *survivors, int64_t n, const sc_camera *cam,
               const sc_opts *opts, sc_splat *splats, sc_window *windows, double *dbg_f64, int32_t *dbg_rect,
               uint8_t *dbg_flags, sc_frame_stats *stats, void *stream)
{
    int rc;
    if ((rc = check_scene(scene)) || (rc = check_camera(cam)) || (rc = check_opts(opts))) return rc;
    if (n < 0 || (n > 0 && (!survivors || !splats || !windows)))
        return fail(SC_ERR_INVALID, "bad survivor / splat / window buffers%s");
    if (!stats) return fail(SC_ERR_INVALID, "stats is NULL%s");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SC_TRY(cudaMemsetAsync(stats, 0, sizeof(sc_frame_stats), st), "memset stats");
    SC_TRY(sc::launch_project(*scene, survivors, nullptr, n, *cam, *opts, splats, windows, nullptr, nullptr, nullptr,
                              nullptr, dbg_f64, dbg_rect, dbg_flags, stats, nullptr, nullptr, st),
           "project");
    return SC_OK;
}

int sc_bin_sort(const sc_scene *scene, const sc_survivor *survivors, int64_t n, const sc_camera *cam,
                const sc_opts *opts, const sc_workspace *ws, sc_splat *splats, sc_window *windows,
                uint32_t *entry_idx, uint32_t *tile_offsets, uint32_t *order_idx, sc_frame_stats *stats,
                void *stream)
{
    int rc;
    if ((rc = check_scene(scene)) || (rc = check_camera(cam)) || (rc = check_opts(opts))) return rc;
    if (!stats || !splats) return fail(SC_ERR_INVALID, "stats / splats are NULL%s");
    if (n < 0 || (n > 0 && !survivors)) return fail(SC_ERR_INVALID, "bad survivor buffer%s");
    sc::Ws w;
    if ((rc = carve(ws, cam->width, cam->height, opts->tile_size, w))) return rc;
    if (n > w.capS) return fail(SC_ERR_INVALID, "n exceeds workspace cap_survivors%s");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    sc_window *wins = windows ? windows : w.wins;
    SC_TRY(cudaMemsetAsync(stats, 0, sizeof(sc_frame_stats), st), "memset stats");
    SC_TRY(cudaMemsetAsync(w.ctr, 0, sizeof(sc::Counters), st), "memset counters");
    uint32_t *order = nullptr, *entries = nullptr;
    SC_TRY(sc::launch_project(*scene, survivors, nullptr, n, *cam, *opts, splats, wins, w.depth64, w.rect, nullptr,
                              nullptr, nullptr, nullptr, nullptr, stats, w.ctr, w.key_b, st),
           "project");
    // reference tile binning (bin_tiles semantics) for parity with the oracle; the order is
    // extracted into order_idx inside (its buffer is reused by the entry sort)
    SC_TRY(sc::launch_bin(w, *scene, survivors, nullptr, n, *cam, wins, stats, false, &order, &entries, nullptr,
                          n > 0 ? order_idx : nullptr, st),
           "bin/sort");
    if (entry_idx) SC_TRY(sc::copy_counted(entries, entry_idx, &w.ctr->entries_eff, w.capE, 1, st), "copy entries");
    if (tile_offsets)
        SC_TRY(cudaMemcpyAsync(tile_offsets, w.tile_off, 4 * (size_t)(w.n_tiles_ref + 1), cudaMemcpyDeviceToDevice, st),
               "copy tile offsets");
    return SC_OK;
}

int sc_blend(const sc_splat *splats, const sc_window *windows, int64_t n_splats, const uint32_t *entry_idx,
             const uint32_t *tile_offsets, const sc_camera *cam, const sc_opts *opts, const sc_frame_out *out,
             void *stream)
{
    int rc;
    if ((rc = check_camera(cam)) || (rc = check_opts(opts))) return rc;
    if (!out || !out->image || !out->trans || !tile_offsets || n_splats < 0 || (n_splats > 0 && (!splats || !windows)))
        return fail(SC_ERR_INVALID, "input / output buffers are NULL%s");
    if (opts->record_contributions && (!out->contrib_max || !out->contrib_sum))
        return fail(SC_ERR_INVALID, "record_contributions needs contrib_max and contrib_sum%s");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (opts->record_contributions && n_splats > 0)
        SC_TRY(cudaMemsetAsync(out->contrib_max, 0, 4 * (size_t)n_splats, st), "memset contrib_max");
    const sc::BlendLists lists{tile_offsets, entry_idx, nullptr, windows, false, nullptr};
    SC_TRY(sc::launch_blend(splats, lists, *cam, *opts, *out, n_splats, nullptr, st), "blend");
    return SC_OK;
}

int sc_render_composed(const sc_scene *scene, const sc_camera *cam, const sc_opts *opts, const sc_workspace *ws,
                       const sc_frame_out *out, void *stream)
{
    int rc;
    if ((rc = check_scene(scene)) || (rc = check_camera(cam)) || (rc = check_opts(opts)) ||
        (rc = check_frame_out(out, opts)))
        return rc;
    sc::Ws w;
    if ((rc = carve(ws, cam->width, cam->height, opts->tile_size, w)) || (rc = check_fit(scene, ws))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    sc_frame_stats *stats = out->stats;
    auto mark = [&](int i) -> cudaError_t {
        if (out->stage_events && i < out->n_stage_events && out->stage_events[i])
            return cudaEventRecord(static_cast<cudaEvent_t>(out->stage_events[i]), st);
        return cudaSuccess;
    };
    SC_TRY(mark(0), "event");
    SC_TRY(cudaMemsetAsync(stats, 0, sizeof(sc_frame_stats), st), "memset stats");
    SC_TRY(cudaMemsetAsync(w.ctr, 0, sizeof(sc::Counters), st), "memset counters");
    SC_TRY(sc::launch_prep(*scene, *cam, *opts, w, stats, st), "prep");
    SC_TRY(sc::launch_cull(*scene, *cam, *opts, w, w.surv, w.capS, stats, st), "cull");
    SC_TRY(mark(1), "event");
    return frame_tail(scene, cam, opts, w, out, st, mark);
}

int sc_render_survivors(const sc_scene *scene, const sc_survivor *survivors, int64_t n, const sc_camera *cam,
                        const sc_opts *opts, const sc_workspace *ws, const sc_frame_out *out, void *stream)
{
    int rc;
    if ((rc = check_scene(scene)) || (rc = check_camera(cam)) || (rc = check_opts(opts)) ||
        (rc = check_frame_out(out, opts)))
        return rc;
    if (n < 0 || (n > 0 && !survivors)) return fail(SC_ERR_INVALID, "bad survivor buffer%s");
    sc::Ws w;
    if ((rc = carve(ws, cam->width, cam->height, opts->tile_size, w)) || (rc = check_fit(scene, ws))) return rc;
    if (n > w.capS) return fail(SC_ERR_INVALID, "n exceeds workspace cap_survivors%s");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto mark = [&](int i) -> cudaError_t {
        if (out->stage_events && i < out->n_stage_events && out->stage_events[i])
            return cudaEventRecord(static_cast<cudaEvent_t>(out->stage_events[i]), st);
        return cudaSuccess;
    };
    SC_TRY(mark(0), "event");
    SC_TRY(cudaMemsetAsync(out->stats, 0, sizeof(sc_frame_stats), st), "memset stats");
    SC_TRY(cudaMemsetAsync(w.ctr, 0, sizeof(sc::Counters), st), "memset counters");
    // per-instance frames and the depth-key range over every instance (no cull: the
    // injected survivors may come from any instance)
    sc_opts popts = *opts;
    popts.frustum_mode = SC_FRUSTUM_OFF;
    popts.band_y0 = popts.band_y1 = 0;
    SC_TRY(sc::launch_prep(*scene, *cam, popts, w, out->stats, st), "prep");
    if (n > 0)
        SC_TRY(cudaMemcpyAsync(w.surv, survivors, sizeof(sc_survivor) * (size_t)n, cudaMemcpyDeviceToDevice, st),
               "copy survivors");
    SC_LAUNCH(sc::k_set_survivors, 1, 1, 0, st, w.ctr, out->stats, n);
    SC_TRY(cudaGetLastError(), "set survivors");
    SC_TRY(mark(1), "event");
    return frame_tail(scene, cam, opts, w, out, st, mark);
}

int sc_vis_mlp_forward(const sc_vis_weights *w, const float *x, int64_t n, float *logits, void *stream)
{
    if (n < 0 || (n > 0 && (!w || !x || !logits))) return fail(SC_ERR_INVALID, "bad MLP forward arguments%s");
    SC_TRY(sc::launch_vis_mlp(w, x, n, logits, static_cast<cudaStream_t>(stream)), "vis mlp");
    return SC_OK;
}

int sc_visibility_labels_or(const float *contrib_max, int64_t n, uint32_t *label_bits, void *stream)
{
    if (n < 0 || (n > 0 && (!contrib_max || !label_bits))) return fail(SC_ERR_INVALID, "bad label arguments%s");
    SC_TRY(sc::launch_labels_or(contrib_max, n, label_bits, static_cast<cudaStream_t>(stream)), "labels");
    return SC_OK;
}

int sc_encode_features(const float *params, const float *x, int64_t n, uint16_t *features, void *stream)
{
    if (n < 0 || (n > 0 && (!params || !x || !features))) return fail(SC_ERR_INVALID, "bad feature arguments%s");
    SC_TRY(sc::launch_encode_features(params, x, n, features, static_cast<cudaStream_t>(stream)), "features");
    return SC_OK;
}

}  // extern "C"
