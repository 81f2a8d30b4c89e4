// Stage (d): (depth, index) order of the passed splats and tile binning.
//
// Reference: argsort(depth, kind="stable") over passed splats
// (sc/raster.py:319) followed by the counting sort bin_tiles
// (sc/_kernels.py:137-165).  B200 version, all on device, no host sync:
//   1. stable LSD radix sort (4 x 8 bits) of the f32 depth keys of all
//      survivors (non-passed keys are 0xFFFFFFFF and sink to the end); the
//      input is in survivor order, so equal keys stay index-ordered;
//   2. tie-fix: runs of equal f32 keys are re-ordered by (f64 depth, index),
//      which makes the order identical to the reference's f64 argsort;
//   3. per-splat tile counts -> exclusive scan -> entry emission
//      (tile id, survivor index) in depth order;
//   4. stable LSD radix sort of the entries by tile id (2 x 8 bits), i.e.
//      the reference's stable counting sort by tile;
//   5. tile offsets (the reference's `counts` array).
// Every kernel reads its element count from device memory, so the whole
// frame stays asynchronous (and CUDA-graph capturable).
#include <algorithm>

#include "common.cuh"

namespace sc {

// ---------------------------------------------------------------------------
// generic exclusive scan of uint32 (3 phases), n read from device or host
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t dev_count(const unsigned long long *n_dev, int64_t n_host)
{
    return n_dev ? std::min<int64_t>((int64_t)*n_dev, n_host) : n_host;
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t *s_warp, uint32_t &total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = THREADS / 32;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_warp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < NW ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[NW - 1];
    const uint32_t r = (wid ? s_warp[wid - 1] : 0u) + v - x;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *in, const unsigned long long *n_dev,
                                                              int64_t n_host, uint32_t *part)
{
    __shared__ uint32_t s_warp[32];
    const int64_t n = dev_count(n_dev, n_host);
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t sum = 0;
    if (base < n) {
        for (int j = 0; j < kScanItems; j++) {
            const int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
            if (i < n) sum += in[i];
        }
    }
    uint32_t total;
    block_excl_scan<kScanThreads>(sum, s_warp, total);
    if (threadIdx.x == 0) part[blockIdx.x] = total;
}

// single block: exclusive scan of the block partials, total -> *total_out
__global__ void __launch_bounds__(1024) k_scan_partials(uint32_t *part, int64_t nblk, unsigned long long *total_out,
                                                        int64_t *stat_out)
{
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_run;
    if (threadIdx.x == 0) s_run = 0;
    __syncthreads();
    for (int64_t base = 0; base < nblk; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const uint32_t x = i < nblk ? part[i] : 0u;
        uint32_t total;
        const uint32_t e = block_excl_scan<1024>(x, s_warp, total);
        if (i < nblk) part[i] = s_run + e;
        __syncthreads();
        if (threadIdx.x == 0) s_run += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (total_out) *total_out = s_run;
        if (stat_out) *stat_out = (int64_t)s_run;
    }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t *in, uint32_t *out,
                                                            const unsigned long long *n_dev, int64_t n_host,
                                                            const uint32_t *part)
{
    __shared__ uint32_t s_warp[32];
    const int64_t n = dev_count(n_dev, n_host);
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    if (base >= n) return;
    // blocked arrangement: thread t owns items [base + t*16, base + t*16 + 16)
    uint32_t v[kScanItems];
    uint32_t sum = 0;
    const int64_t my = base + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        const int64_t i = my + j;
        v[j] = i < n ? in[i] : 0u;
        sum += v[j];
    }
    uint32_t total;
    uint32_t run = block_excl_scan<kScanThreads>(sum, s_warp, total) + part[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; j++) {
        const int64_t i = my + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
}

static cudaError_t scan_excl(const uint32_t *in, uint32_t *out, const unsigned long long *n_dev, int64_t n_max,
                             uint32_t *part, unsigned long long *total_out, int64_t *stat_out, cudaStream_t st)
{
    const int64_t nblk = std::max<int64_t>(1, (n_max + kScanTile - 1) / kScanTile);
    SC_LAUNCH(k_scan_reduce, (int)nblk, kScanThreads, 0, st, in, n_dev, n_max, part);
    SC_LAUNCH(k_scan_partials, 1, 1024, 0, st, part, nblk, total_out, stat_out);
    SC_LAUNCH(k_scan_down, (int)nblk, kScanThreads, 0, st, in, out, n_dev, n_max, part);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// LSD radix sort pass (8-bit digit), reduce-then-scan, stable.
// hist layout: digit-major [256][nblk] so one exclusive scan yields every
// (digit, block) scatter base.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const uint32_t *keys, const unsigned long long *n_dev,
                                                              int64_t n_host, int shift, uint32_t *hist,
                                                              int64_t nblk)
{
    __shared__ uint32_t h[256];
    const int64_t n = dev_count(n_dev, n_host);
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRadixTile;
    if (base < n) {
#pragma unroll 4
        for (int j = 0; j < kRadixItems; j++) {
            const int64_t i = base + (int64_t)j * kRadixThreads + threadIdx.x;
            if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFFu], 1u);
        }
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(const uint32_t *keys_in, const uint32_t *vals_in,
                                                                 uint32_t *keys_out, uint32_t *vals_out,
                                                                 const unsigned long long *n_dev, int64_t n_host,
                                                                 int shift, const uint32_t *hist_scanned,
                                                                 int64_t nblk)
{
    // Stable local ranking with warp-private digit counters: warp w owns the
    // contiguous slice [w * 512, (w + 1) * 512) of the block's keys (read 32 at
    // a time, coalesced), ranks each round with match_any, and keeps running
    // per-digit counts in its own smem row — no block barrier until the end,
    // where one per-digit prefix over warps and one scan over digits give every
    // key its block-local position.  (Index order = warp-major order, so the
    // ranking is stable.)
    constexpr int kWarps = kRadixThreads / 32;
    constexpr int kPerWarp = kRadixTile / kWarps;
    __shared__ uint32_t s_keys[kRadixTile];
    __shared__ uint32_t s_vals[kRadixTile];
    __shared__ uint32_t s_wcnt[kWarps][256];
    __shared__ uint32_t s_dstart[256];   // block-local start of each digit
    __shared__ uint32_t s_gbase[256];    // global scatter base of each digit
    __shared__ uint32_t s_warp[32];
    const int64_t n = dev_count(n_dev, n_host);
    const int64_t base = (int64_t)blockIdx.x * kRadixTile;
    if (base >= n) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int cnt = (int)std::min<int64_t>(kRadixTile, n - base);
#pragma unroll
    for (int w = 0; w < kWarps; w++) s_wcnt[w][tid] = 0;
    s_gbase[tid] = hist_scanned[(int64_t)tid * nblk + blockIdx.x];

    uint32_t k[kRadixItems], v[kRadixItems], rk[kRadixItems];
#pragma unroll
    for (int j = 0; j < kRadixItems; j++) {
        const int i = wid * kPerWarp + j * 32 + lane;
        k[j] = i < cnt ? keys_in[base + i] : 0u;
        v[j] = i < cnt ? vals_in[base + i] : 0u;
    }
    __syncthreads();
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < kRadixItems; j++) {
        const bool ok = wid * kPerWarp + j * 32 + lane < cnt;
        const uint32_t d = ok ? ((k[j] >> shift) & 0xFFu) : 256u + (uint32_t)lane;   // unique dummy digit
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t r = __popc(peers & lt);
        const uint32_t prev = ok ? s_wcnt[wid][d] : 0u;
        __syncwarp();
        if (ok && r == 0) s_wcnt[wid][d] = prev + __popc(peers);
        __syncwarp();
        rk[j] = prev + r;
    }
    __syncthreads();
    {   // per digit (thread = digit): exclusive prefix over warps, then scan over digits
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const uint32_t c = s_wcnt[w][tid];
            s_wcnt[w][tid] = run;
            run += c;
        }
        uint32_t total;
        s_dstart[tid] = block_excl_scan<kRadixThreads>(run, s_warp, total);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixItems; j++) {
        if (wid * kPerWarp + j * 32 + lane < cnt) {
            const uint32_t d = (k[j] >> shift) & 0xFFu;
            const uint32_t pos = s_dstart[d] + s_wcnt[wid][d] + rk[j];
            s_keys[pos] = k[j];
            s_vals[pos] = v[j];
        }
    }
    __syncthreads();
    // coalesced write-out: consecutive positions of one digit are contiguous in the output
    for (int i = tid; i < cnt; i += kRadixThreads) {
        const uint32_t key = s_keys[i];
        const uint32_t d = (key >> shift) & 0xFFu;
        const uint32_t dst = s_gbase[d] + (uint32_t)i - s_dstart[d];
        keys_out[dst] = key;
        vals_out[dst] = s_vals[i];
    }
}

// Sorts (keys, vals) in place-ish over `bits` low bits; result ends in the
// buffer pointed to by *keys_res / *vals_res (ping-pong).
static cudaError_t radix_sort(uint32_t *ka, uint32_t *va, uint32_t *kb, uint32_t *vb, const unsigned long long *n_dev,
                              int64_t n_max, int bits, uint32_t *hist, uint32_t *part, uint32_t **keys_res,
                              uint32_t **vals_res, cudaStream_t st)
{
    const int64_t nblk = std::max<int64_t>(1, (n_max + kRadixTile - 1) / kRadixTile);
    uint32_t *ki = ka, *vi = va, *ko = kb, *vo = vb;
    for (int shift = 0; shift < bits; shift += 8) {
        SC_LAUNCH(k_radix_hist, (int)nblk, kRadixThreads, 0, st, ki, n_dev, n_max, shift, hist, nblk);
        cudaError_t e = scan_excl(hist, hist, nullptr, 256 * nblk, part, nullptr, nullptr, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_radix_scatter, (int)nblk, kRadixThreads, 0, st, ki, vi, ko, vo, n_dev, n_max, shift, hist, nblk);
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    *keys_res = ki;
    *vals_res = vi;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// depth keys: frame-adaptive 32-bit quantisation of the f64 depth over the
// passed splats' [dmin, dmax] (monotone non-decreasing, so key order agrees
// with f64 order wherever keys differ; equal keys go to the tie-fix).  Much
// finer than an f32 key over the same range, so ties are rare.
// ---------------------------------------------------------------------------
__global__ void k_depth_keys(const double *depth64, const unsigned long long *n_dev, int64_t n_host,
                             const Counters *ctr, uint32_t *keys, uint32_t *vals)
{
    const int64_t n = dev_count(n_dev, n_host);
    const double dmin = __longlong_as_double((long long)~ctr->dmin_inv);
    const double dmax = __longlong_as_double((long long)ctr->dmax);
    constexpr double kTop = 4294967040.0;   // < 0xFFFFFFFF, which marks non-passed splats
    const double scale = (ctr->passed > 0 && dmax > dmin) ? kTop / (dmax - dmin) : 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double d = depth64[k];
        uint32_t key = 0xFFFFFFFFu;
        if (d >= 0.0) key = (uint32_t)fmin(floor((d - dmin) * scale), kTop);
        keys[k] = key;
        vals[k] = (uint32_t)k;
    }
}

// ---------------------------------------------------------------------------
// tie-fix: equal keys -> order by (f64 depth, survivor index)
// ---------------------------------------------------------------------------
__global__ void k_tiefix(const uint32_t *keys, uint32_t *vals, const double *depth64, const unsigned long long *n_dev,
                        int64_t n_host, sc_frame_stats *stats)
{
    const int64_t n = dev_count(n_dev, n_host);
    unsigned long long longest = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t key = keys[i];
        if (i > 0 && keys[i - 1] == key) continue;          // not a run head
        if (i + 1 >= n || keys[i + 1] != key) continue;     // run of length 1
        int64_t e = i + 1;
        while (e < n && keys[e] == key) e++;
        longest = std::max<unsigned long long>(longest, (unsigned long long)(e - i));
        // insertion sort on (depth64[v], v); linear when already ordered
        for (int64_t a = i + 1; a < e; a++) {
            const uint32_t va = vals[a];
            const double da = depth64[va];
            int64_t b = a - 1;
            while (b >= i) {
                const uint32_t vb = vals[b];
                const double db = depth64[vb];
                if (db < da || (db == da && vb < va)) break;
                vals[b + 1] = vb;
                b--;
            }
            vals[b + 1] = va;
        }
    }
    if (longest) atomicMax((unsigned long long *)&stats->max_tie_run, longest);
}

// ---------------------------------------------------------------------------
// entries: per passed splat (depth order) count, scan, emit (tile, survivor)
// ---------------------------------------------------------------------------
// The rect of each splat is gathered once here (depth order) and kept
// contiguous in (rlo, rhi) so the emission pass reads it coalesced.
__global__ void k_entry_count(const uint32_t *order, const ushort4 *rect, const unsigned long long *n_dev,
                              int64_t n_host, uint32_t *cnt, uint32_t *rlo, uint32_t *rhi)
{
    const int64_t n = dev_count(n_dev, n_host);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const ushort4 r = rect[order[k]];
        cnt[k] = (uint32_t)(r.y - r.x) * (uint32_t)(r.w - r.z);
        rlo[k] = (uint32_t)r.x | ((uint32_t)r.y << 16);
        rhi[k] = (uint32_t)r.z | ((uint32_t)r.w << 16);
    }
}

__global__ void k_entry_emit(const uint32_t *order, const uint32_t *rlo, const uint32_t *rhi, const uint32_t *off,
                             const unsigned long long *n_dev, int64_t n_host, int n_tx, uint32_t *ekey,
                             uint32_t *eval, const unsigned long long *e_total, unsigned long long *e_eff, int64_t cap_e,
                             sc_frame_stats *stats)
{
    const int64_t n = dev_count(n_dev, n_host);
    const bool over = (int64_t)*e_total > cap_e;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *e_eff = over ? 0ull : *e_total;
        if (over) atomicOr((unsigned long long *)&stats->overflow, 2ull);
    }
    if (over) return;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t sv = order[k];
        const uint32_t a = rlo[k], b = rhi[k];
        const ushort4 r = make_ushort4(a & 0xFFFF, a >> 16, b & 0xFFFF, b >> 16);
        uint32_t o = off[k];
        for (int y = r.z; y < r.w; y++)
            for (int x = r.x; x < r.y; x++) {
                ekey[o] = (uint32_t)(y * n_tx + x);
                eval[o] = sv;
                o++;
            }
    }
}

// tile_off[t] = first entry index with tile >= t, for t in [0, n_tiles]; and
// each entry's pixel window clipped to its tile, 4 bits per bound
// (x0 | x1 << 4 | y0 << 8 | y1 << 12, tile-relative; x0 > x1 = empty),
// gathered once here so the blend's 8 warps per tile stream 2 bytes per
// entry instead of each re-gathering the window from the splat records.
__global__ void k_tile_offsets(const uint32_t *ekey, const uint32_t *eval, const sc_splat *splats,
                               const unsigned long long *e_dev, int64_t cap_e, int64_t n_tiles, int n_tx,
                               uint32_t *tile_off, uint32_t *ewin)
{
    const int64_t E = std::min<int64_t>((int64_t)*e_dev, cap_e);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= E; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = i > 0 ? (int64_t)ekey[i - 1] : -1;
        const int64_t cur = i < E ? (int64_t)ekey[i] : n_tiles;
        for (int64_t t = prev + 1; t <= cur; t++) tile_off[t] = (uint32_t)i;
        if (i < E) {
            const uint2 w = __ldg(reinterpret_cast<const uint2 *>(reinterpret_cast<const char *>(splats + eval[i]) + 40));
            const int tile = (int)cur, ox = (tile % n_tx) * kTile, oy = (tile / n_tx) * kTile;
            const int x0 = max((int)(int16_t)(w.x & 0xFFFF) - ox, 0), x1 = min((int)(int16_t)(w.x >> 16) - ox, 15);
            const int y0 = max((int)(int16_t)(w.y & 0xFFFF) - oy, 0), y1 = min((int)(int16_t)(w.y >> 16) - oy, 15);
            uint32_t code = 0x000F;   // empty
            if (x0 <= x1 && y0 <= y1) code = (uint32_t)(x0 | (x1 << 4) | (y0 << 8) | (y1 << 12));
            ewin[i] = code;
        }
    }
}

// ---------------------------------------------------------------------------
// per-(tile, 8x4 pixel block) entry lists for the blend: list (t, b) is the
// stable (depth-order) subsequence of tile t's entries whose clipped window
// touches block b (b = 2 row + col: x in [8 col, 8 col + 7], y in [4 row, 4 row + 3]).
// ---------------------------------------------------------------------------
constexpr uint32_t kEmpty = 0x000Fu;   // empty window code (x0 = 15 > x1 = 0)

__device__ __forceinline__ uint32_t code_blocks(uint32_t c)
{
    const uint32_t x0 = c & 15u, x1 = (c >> 4) & 15u, y0 = (c >> 8) & 15u, y1 = (c >> 12) & 15u;
    if (x0 > x1 || y0 > y1) return 0u;
    const uint32_t cols = (x0 <= 7u ? 1u : 0u) | (x1 >= 8u ? 2u : 0u);
    const uint32_t r0 = y0 >> 2, r1 = y1 >> 2;
    uint32_t m = 0u;
#pragma unroll
    for (uint32_t r = 0; r < 4; r++)
        if (r >= r0 && r <= r1) m |= cols << (2 * r);
    return m;
}

__global__ void __launch_bounds__(256) k_block_count(const uint32_t *tile_off, const uint32_t *ewin, uint32_t *bcnt)
{
    __shared__ uint32_t s_cnt[8][8];
    const int tile = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t s = tile_off[tile], e = tile_off[tile + 1];
    uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t i = s + wid * 32u + lane; i - lane < e; i += 256u) {
        const uint32_t m = i < e ? code_blocks(__ldg(ewin + i)) : 0u;
#pragma unroll
        for (int b = 0; b < 8; b++) cnt[b] += __popc(__ballot_sync(0xffffffffu, (m >> b) & 1u));
    }
    if (lane == 0)
#pragma unroll
        for (int b = 0; b < 8; b++) s_cnt[wid][b] = cnt[b];
    __syncthreads();
    if (threadIdx.x < 8) {
        uint32_t t = 0;
        for (int w = 0; w < 8; w++) t += s_cnt[w][threadIdx.x];
        bcnt[8 * (size_t)tile + threadIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) k_block_fill(const uint32_t *tile_off, const uint32_t *ewin,
                                                    const uint32_t *entry_idx, uint32_t *boff, int64_t n_tiles,
                                                    uint32_t *lidx, uint32_t *lcode, int64_t cap_l, Counters *ctr,
                                                    sc_frame_stats *stats)
{
    __shared__ uint32_t s_cnt[8][8];   // [warp][block]: members in this chunk -> exclusive prefix
    __shared__ uint32_t s_pos[8];      // next output position of each block list
    const int tile = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned long long total = ctr->block_entries;
    const bool ok = total <= (unsigned long long)cap_l;
    if (blockIdx.x == 0 && tid == 0) {
        ctr->lists_ok = ok ? 1ull : 0ull;
        boff[8 * n_tiles] = (uint32_t)total;
        stats->block_entries = (int64_t)total;
        if (!ok) atomicOr((unsigned long long *)&stats->overflow, 4ull);
    }
    if (!ok) return;
    const uint32_t s = tile_off[tile], e = tile_off[tile + 1];
    if (tid < 8) s_pos[tid] = boff[8 * (size_t)tile + tid];
    const uint32_t lt = lanemask_lt();
    uint32_t i = s + tid;
    uint32_t c = kEmpty, v = 0u;
    if (i < e) {
        c = __ldg(ewin + i);
        v = __ldg(entry_idx + i);
    }
    for (uint32_t chunk = s; chunk < e; chunk += 256u, i += 256u) {
        // prefetch the next chunk while this one is ranked
        uint32_t nc = kEmpty, nv = 0u;
        if (i + 256u < e) {
            nc = __ldg(ewin + i + 256u);
            nv = __ldg(entry_idx + i + 256u);
        }
        const uint32_t m = i < e ? code_blocks(c) : 0u;
        uint32_t bal[8];
#pragma unroll
        for (int b = 0; b < 8; b++) bal[b] = __ballot_sync(0xffffffffu, (m >> b) & 1u);
        if (lane == 0)
#pragma unroll
            for (int b = 0; b < 8; b++) s_cnt[wid][b] = __popc(bal[b]);
        __syncthreads();
        if (tid < 8) {
            uint32_t run = s_pos[tid];
            for (int w = 0; w < 8; w++) {
                const uint32_t k = s_cnt[w][tid];
                s_cnt[w][tid] = run;
                run += k;
            }
            s_pos[tid] = run;
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < 8; b++) {
            if ((m >> b) & 1u) {
                const uint32_t pos = s_cnt[wid][b] + __popc(bal[b] & lt);
                lidx[pos] = v;
                lcode[pos] = c;
            }
        }
        __syncthreads();
        c = nc;
        v = nv;
    }
}

static int grid_for(int64_t n, int threads)
{
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)nsm * 16));
}

// n_dev: survivor count (device).  Inputs: ws.key_a / val_a / depth64 / rect
// from the projection.  Outputs: order (passed survivors by (depth, index)),
// entries (survivor index per entry, tile-major), ws.tile_off, stats.entries.
cudaError_t launch_bin(const Ws &ws, const unsigned long long *n_dev, int64_t n_max, const sc_camera &cam,
                       const sc_splat *splats, sc_frame_stats *stats, uint32_t **order_out, uint32_t **entries_out,
                       uint32_t **win_out, cudaStream_t st)
{
    cudaError_t e;
    uint32_t *keys_s = nullptr, *order = nullptr;
    SC_LAUNCH(k_depth_keys, grid_for(n_max, 256), 256, 0, st, ws.depth64, n_dev, n_max, ws.ctr, ws.key_a, ws.val_a);
    e = radix_sort(ws.key_a, ws.val_a, ws.key_b, ws.val_b, n_dev, n_max, 32, ws.hist, ws.scan_part, &keys_s, &order,
                   st);
    if (e != cudaSuccess) return e;
    const unsigned long long *p_dev = &ws.ctr->passed;   // passed splats lead the sorted order
    SC_LAUNCH(k_tiefix, grid_for(n_max, 256), 256, 0, st, keys_s, order, ws.depth64, p_dev, n_max, stats);
    // both key buffers are free once the tie-fix is done: depth-ordered rects
    uint32_t *rlo = ws.key_a, *rhi = ws.key_b;
    SC_LAUNCH(k_entry_count, grid_for(n_max, 256), 256, 0, st, order, ws.rect, p_dev, n_max, ws.ecount, rlo, rhi);
    e = scan_excl(ws.ecount, ws.ecount, p_dev, n_max, ws.scan_part, &ws.ctr->entries, &stats->entries, st);
    if (e != cudaSuccess) return e;
    SC_LAUNCH(k_entry_emit, grid_for(n_max, 256), 256, 0, st, order, rlo, rhi, ws.ecount, p_dev, n_max, ws.n_tx,
              ws.ekey_a, ws.eval_a, &ws.ctr->entries, &ws.ctr->entries_eff, ws.capE, stats);
    int bits = 0;
    while ((1ll << bits) < ws.n_tiles) bits += 8;
    uint32_t *ek = nullptr, *ev = nullptr;
    if (bits == 0) bits = 8;
    e = radix_sort(ws.ekey_a, ws.eval_a, ws.ekey_b, ws.eval_b, &ws.ctr->entries_eff, ws.capE, bits, ws.hist,
                   ws.scan_part, &ek, &ev, st);
    if (e != cudaSuccess) return e;
    // the ping-pong key buffer not holding the sorted keys is free: window stream
    uint32_t *ewin = (ek == ws.ekey_a) ? ws.ekey_b : ws.ekey_a;
    SC_LAUNCH(k_tile_offsets, grid_for(ws.capE + 1, 256), 256, 0, st, ek, ev, splats, &ws.ctr->entries_eff, ws.capE,
              ws.n_tiles, ws.n_tx, ws.tile_off, ewin);
    // the blend's per-(tile, 8x4 block) lists: count, scan, stable fill
    SC_LAUNCH(k_block_count, (int)ws.n_tiles, 256, 0, st, ws.tile_off, ewin, ws.boff);
    e = scan_excl(ws.boff, ws.boff, nullptr, 8 * ws.n_tiles, ws.scan_part, &ws.ctr->block_entries, nullptr, st);
    if (e != cudaSuccess) return e;
    SC_LAUNCH(k_block_fill, (int)ws.n_tiles, 256, 0, st, ws.tile_off, ewin, ev, ws.boff, ws.n_tiles, ws.lidx, ws.lcode,
              ws.capL, ws.ctr, stats);
    *order_out = order;
    *entries_out = ev;
    if (win_out) *win_out = ewin;
    return cudaGetLastError();
}

}  // namespace sc
