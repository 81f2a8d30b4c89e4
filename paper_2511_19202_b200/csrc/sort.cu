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
// Sorts on key bits [bit_lo, bit_hi) (8-bit digits; bits below bit_lo ride along unsorted).
static cudaError_t radix_sort(uint32_t *ka, uint32_t *va, uint32_t *kb, uint32_t *vb, const unsigned long long *n_dev,
                              int64_t n_max, int bit_lo, int bit_hi, uint32_t *hist, uint32_t *part,
                              uint32_t **keys_res, uint32_t **vals_res, cudaStream_t st)
{
    const int64_t nblk = std::max<int64_t>(1, (n_max + kRadixTile - 1) / kRadixTile);
    uint32_t *ki = ka, *vi = va, *ko = kb, *vo = vb;
    for (int shift = bit_lo; shift < bit_hi; shift += 8) {
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

// tile_off[t] = first entry index with tile >= t, for t in [0, n_tiles] (the
// reference's `counts`; stage-level API only)
__global__ void k_tile_offsets(const uint32_t *ekey, const unsigned long long *e_dev, int64_t cap_e, int64_t n_tiles,
                               uint32_t *tile_off)
{
    const int64_t E = std::min<int64_t>((int64_t)*e_dev, cap_e);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= E; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = i > 0 ? (int64_t)ekey[i - 1] : -1;
        const int64_t cur = i < E ? (int64_t)ekey[i] : n_tiles;
        for (int64_t t = prev + 1; t <= cur; t++) tile_off[t] = (uint32_t)i;
    }
}

// ---------------------------------------------------------------------------
// Frame-path binning: 8x4 pixel blocks instead of 16x16 tiles.
//
// Each passed splat (in depth order) emits one entry per 8x4 block its pixel
// window touches; block b of tile t has id 8 t + b (b = 2 row + col: x in
// [8 col, 8 col + 7], y in [4 row, 4 row + 3]), so a tile's blocks are
// contiguous.  The sort key is id << 10 | the window clipped to the block
// (x0 | x1 << 3 | y0 << 6 | y1 << 8, block-relative); the radix sort only
// sorts the id bits, so the clipped window rides along.  Being a stable sort
// of the depth-ordered emission, block list (t, b) is exactly the depth-order
// subsequence of the reference's tile-t entry list whose window touches
// block b (the only entries the reference composites onto those pixels):
// one blend warp walks one list.
// ---------------------------------------------------------------------------
constexpr int kCodeBits = 10;

__global__ void k_bentry_count(const uint32_t *order, const sc_window *wins, const unsigned long long *n_dev,
                               int64_t n_host, int width, int height, uint32_t *cnt, uint32_t *wlo, uint32_t *whi)
{
    const int64_t n = dev_count(n_dev, n_host);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const uint2 w = __ldg(reinterpret_cast<const uint2 *>(wins + order[k]));
        // pixels outside the image are never composited (reference th/tw clamp)
        const int x0 = max((int)(int16_t)(w.x & 0xFFFF), 0), x1 = min((int)(int16_t)(w.x >> 16), width - 1);
        const int y0 = max((int)(int16_t)(w.y & 0xFFFF), 0), y1 = min((int)(int16_t)(w.y >> 16), height - 1);
        uint32_t c = 0;
        if (x0 <= x1 && y0 <= y1) {
            c = (uint32_t)((x1 / 8 - x0 / 8 + 1) * (y1 / 4 - y0 / 4 + 1));
            wlo[k] = (uint32_t)x0 | ((uint32_t)x1 << 16);
            whi[k] = (uint32_t)y0 | ((uint32_t)y1 << 16);
        } else {   // canonical empty window: the emission recomputes the count from these
            wlo[k] = 1u;
            whi[k] = 1u;
        }
        cnt[k] = c;
    }
}

__global__ void k_bentry_emit(const uint32_t *order, const uint32_t *wlo, const uint32_t *whi, const uint32_t *off,
                              const unsigned long long *n_dev, int64_t n_host, int n_tx, uint32_t *ekey,
                              uint32_t *eval, const unsigned long long *e_total, unsigned long long *e_eff,
                              int64_t cap_e, sc_frame_stats *stats)
{
    const int64_t n = dev_count(n_dev, n_host);
    const bool over = (int64_t)*e_total > cap_e;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *e_eff = over ? 0ull : *e_total;
        stats->block_entries = (int64_t)*e_total;
        if (over) atomicOr((unsigned long long *)&stats->overflow, 2ull);
    }
    if (over) return;
    // Warp-cooperative, load-balanced: a warp owns 32 consecutive splats and
    // emits their (contiguous) entries 32 at a time, lane l producing output
    // o = step + l; the owning splat is found by an upper-bound search over the
    // warp's exclusive counts (5 shuffles).  Splats covering thousands of
    // blocks (close to the camera) no longer serialise one thread, and the
    // stores are coalesced.
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 32; base < n; base += n_warps * 32) {
        const int64_t k = base + lane;
        int x0 = 1, x1 = 0, y0 = 1, y1 = 0;
        uint32_t sv = 0;
        if (k < n) {
            const uint32_t a = wlo[k], b = whi[k];
            x0 = (int)(a & 0xFFFF);
            x1 = (int)(a >> 16);
            y0 = (int)(b & 0xFFFF);
            y1 = (int)(b >> 16);
            sv = order[k];
        }
        const uint32_t cnt = (x0 <= x1 && y0 <= y1) ? (uint32_t)((x1 / 8 - x0 / 8 + 1) * (y1 / 4 - y0 / 4 + 1)) : 0u;
        uint32_t incl = cnt;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, s);
            if (lane >= s) incl += y;
        }
        const uint32_t excl = incl - cnt;
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t obase = __shfl_sync(0xffffffffu, off[base], 0);
        for (uint32_t o0 = 0; o0 < total; o0 += 32) {
            const uint32_t o = o0 + lane;
            int s = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t e = __shfl_sync(0xffffffffu, excl, s + step);
                if (e <= o) s += step;
            }
            const uint32_t li = o - __shfl_sync(0xffffffffu, excl, s);
            const int X0 = __shfl_sync(0xffffffffu, x0, s), X1 = __shfl_sync(0xffffffffu, x1, s);
            const int Y0 = __shfl_sync(0xffffffffu, y0, s), Y1 = __shfl_sync(0xffffffffu, y1, s);
            const uint32_t v = __shfl_sync(0xffffffffu, sv, s);
            if (o < total) {
                const int w = X1 / 8 - X0 / 8 + 1;
                const int bx = X0 / 8 + (int)(li % (uint32_t)w), by = Y0 / 4 + (int)(li / (uint32_t)w);
                const int rx0 = max(X0 - 8 * bx, 0), rx1 = min(X1 - 8 * bx, 7);
                const int ry0 = max(Y0 - 4 * by, 0), ry1 = min(Y1 - 4 * by, 3);
                const uint32_t id = (uint32_t)(((by >> 2) * n_tx + (bx >> 1)) * 8 + (by & 3) * 2 + (bx & 1));
                ekey[obase + o] = (id << kCodeBits) | (uint32_t)(rx0 | (rx1 << 3) | (ry0 << 6) | (ry1 << 8));
                eval[obase + o] = v;
            }
        }
    }
}

// boff[b] = first entry with block id >= b, for b in [0, n_blocks]
__global__ void k_block_offsets(const uint32_t *ekey, const unsigned long long *e_dev, int64_t cap_e,
                                int64_t n_blocks, uint32_t *boff)
{
    const int64_t E = std::min<int64_t>((int64_t)*e_dev, cap_e);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= E; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = i > 0 ? (int64_t)(ekey[i - 1] >> kCodeBits) : -1;
        const int64_t cur = i < E ? (int64_t)(ekey[i] >> kCodeBits) : n_blocks;
        for (int64_t t = prev + 1; t <= cur; t++) boff[t] = (uint32_t)i;
    }
}

static int grid_for(int64_t n, int threads)
{
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)nsm * 16));
}

static int bits_for(int64_t n)
{
    int b = 0;
    while ((1ll << b) < n) b++;
    return b;
}

// n_dev: survivor count (device).  Inputs: ws.depth64 / rect and the splat
// records from the projection.  Always: order = passed survivors by (depth,
// index).  blocks = true (frame path): block lists (entries_out = survivor per
// entry, keys_out = id << 10 | window, ws.boff).  blocks = false (stage-level
// API, parity with the reference): tile entries and ws.tile_off, exactly
// bin_tiles' output.
cudaError_t launch_bin(const Ws &ws, const unsigned long long *n_dev, int64_t n_max, const sc_camera &cam,
                       const sc_window *wins, sc_frame_stats *stats, bool blocks, uint32_t **order_out,
                       uint32_t **entries_out, uint32_t **keys_out, cudaStream_t st)
{
    cudaError_t e;
    uint32_t *keys_s = nullptr, *order = nullptr;
    SC_LAUNCH(k_depth_keys, grid_for(n_max, 256), 256, 0, st, ws.depth64, n_dev, n_max, ws.ctr, ws.key_a, ws.val_a);
    e = radix_sort(ws.key_a, ws.val_a, ws.key_b, ws.val_b, n_dev, n_max, 0, 32, ws.hist, ws.scan_part, &keys_s, &order,
                   st);
    if (e != cudaSuccess) return e;
    const unsigned long long *p_dev = &ws.ctr->passed;   // passed splats lead the sorted order
    SC_LAUNCH(k_tiefix, grid_for(n_max, 256), 256, 0, st, keys_s, order, ws.depth64, p_dev, n_max, stats);
    // both key buffers are free once the tie-fix is done: depth-ordered rects / windows
    uint32_t *rlo = ws.key_a, *rhi = ws.key_b;
    uint32_t *ek = nullptr, *ev = nullptr;
    if (blocks) {
        SC_LAUNCH(k_bentry_count, grid_for(n_max, 256), 256, 0, st, order, wins, p_dev, n_max, cam.width, cam.height,
                  ws.ecount, rlo, rhi);
        e = scan_excl(ws.ecount, ws.ecount, p_dev, n_max, ws.scan_part, &ws.ctr->entries, nullptr, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_bentry_emit, grid_for(n_max, 256), 256, 0, st, order, rlo, rhi, ws.ecount, p_dev, n_max, ws.n_tx,
                  ws.ekey_a, ws.eval_a, &ws.ctr->entries, &ws.ctr->entries_eff, ws.capE, stats);
        const int64_t n_blocks = 8 * ws.n_tiles;
        e = radix_sort(ws.ekey_a, ws.eval_a, ws.ekey_b, ws.eval_b, &ws.ctr->entries_eff, ws.capE, kCodeBits,
                       kCodeBits + bits_for(n_blocks), ws.hist, ws.scan_part, &ek, &ev, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_block_offsets, grid_for(ws.capE + 1, 256), 256, 0, st, ek, &ws.ctr->entries_eff, ws.capE, n_blocks,
                  ws.boff);
    } else {
        SC_LAUNCH(k_entry_count, grid_for(n_max, 256), 256, 0, st, order, ws.rect, p_dev, n_max, ws.ecount, rlo, rhi);
        e = scan_excl(ws.ecount, ws.ecount, p_dev, n_max, ws.scan_part, &ws.ctr->entries, &stats->entries, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_entry_emit, grid_for(n_max, 256), 256, 0, st, order, rlo, rhi, ws.ecount, p_dev, n_max, ws.n_tx,
                  ws.ekey_a, ws.eval_a, &ws.ctr->entries, &ws.ctr->entries_eff, ws.capE, stats);
        e = radix_sort(ws.ekey_a, ws.eval_a, ws.ekey_b, ws.eval_b, &ws.ctr->entries_eff, ws.capE, 0,
                       std::max(1, bits_for(ws.n_tiles)), ws.hist, ws.scan_part, &ek, &ev, st);
        if (e != cudaSuccess) return e;
        SC_LAUNCH(k_tile_offsets, grid_for(ws.capE + 1, 256), 256, 0, st, ek, &ws.ctr->entries_eff, ws.capE,
                  ws.n_tiles, ws.tile_off);
    }
    *order_out = order;
    *entries_out = ev;
    if (keys_out) *keys_out = ek;
    return cudaGetLastError();
}

}  // namespace sc
