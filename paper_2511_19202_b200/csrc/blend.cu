// Stage (e): per-tile front-to-back alpha blending.
//
// Reference: composite_tiles (sc/_kernels.py:190-275) + finish()
// (sc/raster.py:267-282).  Semantics per pixel are the reference's: walk the
// tile's entries in (depth, index) order, skip splats with alpha0 < 1/255,
// composite inside the splat's exact f64 pixel window when
// p_min <= power <= 0, alpha = min(0.99, alpha0 e^power), retire the pixel
// after compositing once T < stop_transmittance.  fp32 arithmetic
// (tolerance stated in tests/test_gpu_parity.py).
//
// B200 mapping — every warp is an independent worker with no CTA barrier:
//   * a warp owns an 8x4 pixel block (lane = 8 row + col) of one 16x16 tile;
//     a CTA is 4 warps = half a tile, and CTAs are dispatched heaviest tile
//     first (LPT order by log2 entry count, k_tile_order) so the long
//     silhouette tiles of a 100M-Gaussian frame start at once instead of
//     forming the tail;
//   * the warp walks its tile's entry list 128 entries at a time: entry
//     indices (coalesced) and the 8-byte pixel windows (gather) of the NEXT
//     128 are prefetched into registers while the current 128 are blended;
//   * an entry is processed only when its window intersects the warp's ALIVE
//     pixels (32-bit footprint mask vs ballot of live lanes), so saturated
//     pixels cost nothing; the lanes that hit load their entry's 48-byte
//     record and the warp broadcasts each hit's fields with shuffles;
//   * a warp exits when its 32 pixels have retired.
// The first version staged 256-entry batches in shared memory behind a CTA
// barrier; ncu showed the barrier stall dominating (warps with silhouette
// pixels held the other seven) and one SM busy for the whole kernel.
#include <algorithm>

#include "common.cuh"

namespace sc {

#ifdef SC_BLEND_STATS
// instrumented build only (libsplatcull_b200_dbg.so): per tile
// [entries, entry slots walked, (entry, warp) hits, pixel evaluations, max warp cycles, 0, 0, 0]
constexpr int kDbgTiles = 32400;
__device__ unsigned long long g_blend_dbg[kDbgTiles * 8];
#endif

constexpr int kBlendWarps = 8;              // warps per CTA (one 16x16 tile)
constexpr int kSlots = 4;                   // 32-entry slots per prefetch group

// 32-bit footprint of window w on the 8x4 block at (bx0, by0)
__device__ __forceinline__ uint32_t block_mask(int x0, int x1, int y0, int y1, int bx0, int by0)
{
    const int lo = max(x0, bx0), hi = min(x1, bx0 + 7);
    const int rlo = max(y0, by0), rhi = min(y1, by0 + 3);
    if (lo > hi || rlo > rhi) return 0u;
    const uint32_t cols = (0xFFu >> (7 - (hi - bx0))) & (0xFFu << (lo - bx0));
    const uint32_t rows = (0x01010101u << (8 * (rlo - by0))) & (0x01010101u >> (8 * (3 - (rhi - by0))));
    return cols * rows;
}

// 32x32 bit-matrix transpose across a warp: lane r holds row r on entry and
// column r on exit (bit c of the result = bit r of lane c's input).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane)
{
    constexpr uint32_t kMask[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0, j = 16; s < 5; s++, j >>= 1) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~kMask[s]) | ((y >> j) & kMask[s])) : ((x & kMask[s]) | ((y << j) & ~kMask[s]));
    }
    return x;
}

__device__ __forceinline__ int lo16(uint32_t w) { return (int)(int16_t)(w & 0xFFFFu); }
__device__ __forceinline__ int hi16(uint32_t w) { return (int)(int16_t)(w >> 16); }

__global__ void __launch_bounds__(kBlendWarps * 32) k_blend(const sc_splat *__restrict__ splats, int64_t n_splats,
                                                            const uint32_t *__restrict__ entry_idx,
                                                            const uint32_t *__restrict__ tile_off,
                                                            const uint16_t *__restrict__ ewin,
                                                            const uint32_t *__restrict__ task_order, int width,
                                                            int height, int n_tx, float stop_t, float bg_r,
                                                            float bg_g, float bg_b, int record, float *image,
                                                            float *trans, float *csum, float *cmax)
{
    const int tile = (int)(task_order ? task_order[blockIdx.x] : blockIdx.x);
    const int tyi = tile / n_tx, txi = tile - tyi * n_tx;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ox = txi * kTile, oy = tyi * kTile;              // tile origin
    const int bx0 = (wid & 1) * 8, by0 = (wid >> 1) * 4;        // warp block, tile-relative
    const int px = ox + bx0 + (lane & 7), py = oy + by0 + (lane >> 3);
    const bool inside = px < width && py < height;
    const float fpx = (float)px, fpy = (float)py;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, cs = 0.0f;
    bool done = !inside;
    const uint32_t start = tile_off[tile], end = tile_off[tile + 1];
    const char *rec = reinterpret_cast<const char *>(splats);
#ifdef SC_BLEND_STATS
    unsigned long long d_slots = 0, d_hits = 0, d_evals = 0, d_iters = 0;
    const long long d_t0 = clock64();
#endif

    // per lane, slot k of the current group: entry base + 32 k + lane.
    // code = tile-relative window x0 | x1 << 4 | y0 << 8 | y1 << 12 (x0 > x1: empty)
    uint32_t code[kSlots], ncode[kSlots], idx[kSlots], nidx[kSlots];
    auto prefetch = [&](uint32_t base, uint32_t *pc, uint32_t *pi) {
#pragma unroll
        for (int k = 0; k < kSlots; k++) {
            const uint32_t e = base + 32u * k + lane;
            pc[k] = 0x000Fu;
            pi[k] = 0xFFFFFFFFu;
            if (e < end) {
                if (ewin) {           // entry-aligned stream: 2 bytes, coalesced; index loaded on a hit
                    pc[k] = __ldg(ewin + e);
                } else {
                    uint32_t s = __ldg(entry_idx + e);
                    pi[k] = (int64_t)s < n_splats ? s : 0xFFFFFFFFu;
                }
            }
        }
        if (!ewin) {
#pragma unroll
            for (int k = 0; k < kSlots; k++) {
                if (pi[k] == 0xFFFFFFFFu) continue;
                const uint2 w = __ldg(reinterpret_cast<const uint2 *>(rec + 48 * (size_t)pi[k] + 40));
                const int x0 = max(lo16(w.x) - ox, 0), x1 = min(hi16(w.x) - ox, 15);
                const int y0 = max(lo16(w.y) - oy, 0), y1 = min(hi16(w.y) - oy, 15);
                if (x0 <= x1 && y0 <= y1) pc[k] = (uint32_t)(x0 | (x1 << 4) | (y0 << 8) | (y1 << 12));
            }
        }
    };

    if (!__all_sync(0xffffffffu, done) && start < end) {
        prefetch(start, code, idx);
        for (uint32_t base = start; base < end; base += 32u * kSlots) {
            const bool more = base + 32u * kSlots < end;
            if (more) prefetch(base + 32u * kSlots, ncode, nidx);
#pragma unroll
            for (int k = 0; k < kSlots; k++) {
                const uint32_t alive = __ballot_sync(0xffffffffu, !done);
                if (!alive) break;
                // footprint of this lane's entry on the warp's alive pixels
                const uint32_t c = code[k];
                const uint32_t fp =
                    block_mask(c & 15u, (c >> 4) & 15u, (c >> 8) & 15u, c >> 12, bx0, by0) & alive;
#ifdef SC_BLEND_STATS
                d_slots++;
#endif
                if (!__any_sync(0xffffffffu, fp != 0u)) continue;
                float4 ga = make_float4(0.f, 0.f, 0.f, 0.f), pa = ga;
                float2 gb2 = make_float2(0.f, 0.f);
                if (fp) {
                    if (ewin) {
                        const uint32_t s = __ldg(entry_idx + base + 32u * k + lane);
                        idx[k] = (int64_t)s < n_splats ? s : 0u;
                    }
                    const float4 *src = reinterpret_cast<const float4 *>(rec + 48 * (size_t)idx[k]);
                    ga = __ldg(src);
                    pa = __ldg(src + 1);
                    gb2 = __ldg(reinterpret_cast<const float2 *>(src + 2));
                }
#ifdef SC_BLEND_STATS
                d_hits += __popc(__ballot_sync(0xffffffffu, fp != 0u)) * (lane == 0);
#endif
                // 32x32 bit transpose: bit j of `mine` = entry (slot lane) j covers my pixel
                uint32_t mine = transpose32(fp, lane);
                // each lane walks its own entries in order; the warp iterates
                // max-over-lanes times (fields fetched from lane j by shuffle)
                while (__any_sync(0xffffffffu, mine != 0u)) {
                    const bool act = mine != 0u;
                    const int srcl = act ? __ffs(mine) - 1 : lane;
                    mine &= mine - 1u;
                    const float mx = __shfl_sync(0xffffffffu, ga.x, srcl);
                    const float my = __shfl_sync(0xffffffffu, ga.y, srcl);
                    const float ha = __shfl_sync(0xffffffffu, ga.z, srcl);
                    const float hb = __shfl_sync(0xffffffffu, ga.w, srcl);
                    const float hc = __shfl_sync(0xffffffffu, pa.x, srcl);
                    const float op = __shfl_sync(0xffffffffu, pa.y, srcl);
                    const float pmin = __shfl_sync(0xffffffffu, pa.z, srcl);
                    const float c0 = __shfl_sync(0xffffffffu, pa.w, srcl);
                    const float c1 = __shfl_sync(0xffffffffu, gb2.x, srcl);
                    const float c2 = __shfl_sync(0xffffffffu, gb2.y, srcl);
                    const uint32_t sidx = record ? __shfl_sync(0xffffffffu, idx[k], srcl) : 0u;
#ifdef SC_BLEND_STATS
                    d_evals += act;
                    d_iters += (lane == 0);
#endif
                    if (act) {
                        const float dx = fpx - mx, dy = fpy - my;
                        const float power = -(ha * dx * dx + hc * dy * dy) - hb * dx * dy;
                        if (!(power > 0.0f || power < pmin)) {
                            const float alpha = fminf(0.99f, op * __expf(power));
                            const float contrib = alpha * T;
                            cr += contrib * c0;
                            cg += contrib * c1;
                            cb += contrib * c2;
                            T = T * (1.0f - alpha);
                            if (record) {
                                cs += contrib;
                                if (contrib > 0.0f) atomicMax(reinterpret_cast<int *>(cmax) + sidx, __float_as_int(contrib));
                            }
                            if (T < stop_t) {
                                done = true;
                                mine = 0u;
                            }
                        }
                    }
                }
            }
            if (__all_sync(0xffffffffu, done) || !more) break;
#pragma unroll
            for (int k = 0; k < kSlots; k++) {
                idx[k] = nidx[k];
                code[k] = ncode[k];
            }
        }
    }
#ifdef SC_BLEND_STATS
    for (int o = 16; o > 0; o >>= 1) d_evals += __shfl_down_sync(0xffffffffu, d_evals, o);
    if (tile < kDbgTiles && lane == 0) {
        unsigned long long *dd = g_blend_dbg + 8 * (size_t)tile;
        dd[0] = end - start;
        atomicAdd(dd + 1, d_slots);
        atomicAdd(dd + 2, d_hits);
        atomicAdd(dd + 3, d_evals);
        atomicMax(dd + 4, (unsigned long long)(clock64() - d_t0));
        atomicAdd(dd + 5, d_iters);
    }
#endif
    if (inside) {
        const int64_t p = (int64_t)py * width + px;
        image[3 * p + 0] = cr + T * bg_r;
        image[3 * p + 1] = cg + T * bg_g;
        image[3 * p + 2] = cb + T * bg_b;
        trans[p] = T;
        if (record && csum) csum[p] = cs;
    }
}

// LPT dispatch order: heavier tiles first (bucketed by floor(log2(entries));
// the order inside a bucket is irrelevant to the result).
__global__ void __launch_bounds__(1024) k_tile_order(const uint32_t *tile_off, int64_t n_tiles, uint32_t *order)
{
    __shared__ uint32_t hist[33], base[33];
    if (threadIdx.x < 33) hist[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint32_t c = tile_off[t + 1] - tile_off[t];
        atomicAdd(&hist[c ? 32 - __clz(c) : 0], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 32; b >= 0; b--) {
            base[b] = run;
            run += hist[b];
        }
    }
    __syncthreads();
    for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) {
        const uint32_t c = tile_off[t + 1] - tile_off[t];
        order[atomicAdd(&base[c ? 32 - __clz(c) : 0], 1u)] = (uint32_t)t;
    }
}

__global__ void k_count_used(const float *cmax, const unsigned long long *n_dev, int64_t n_host,
                             sc_frame_stats *stats)
{
    const int64_t n = n_dev ? std::min<int64_t>((int64_t)*n_dev, n_host) : n_host;
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += cmax[i] > 0.0f;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long *)&stats->used, c);
}

cudaError_t launch_blend(const sc_splat *splats, const uint32_t *entry_idx, const uint32_t *tile_off,
                         const uint16_t *ewin, const sc_camera &cam, const sc_opts &opts,
                         const sc_frame_out &out, int64_t n_splats, uint32_t *task_order, cudaStream_t st)
{
    const int n_tx = (cam.width + kTile - 1) / kTile, n_ty = (cam.height + kTile - 1) / kTile;
    const int64_t n_tiles = (int64_t)n_tx * n_ty;
    if (task_order) SC_LAUNCH(k_tile_order, 1, 1024, 0, st, tile_off, n_tiles, task_order);
    SC_LAUNCH(k_blend, (int)n_tiles, kBlendWarps * 32, 0, st, splats, n_splats, entry_idx, tile_off, ewin, task_order,
              cam.width, cam.height, n_tx, (float)opts.stop_transmittance, (float)opts.background[0],
              (float)opts.background[1], (float)opts.background[2], opts.record_contributions ? 1 : 0, out.image,
              out.trans, out.contrib_sum, out.contrib_max);
    return cudaGetLastError();
}

cudaError_t launch_count_used(const float *cmax, const unsigned long long *n_dev, int64_t n_max,
                              sc_frame_stats *stats, cudaStream_t st)
{
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_max + 255) / 256, (int64_t)nsm * 8));
    SC_LAUNCH(k_count_used, grid, 256, 0, st, cmax, n_dev, n_max, stats);
    return cudaGetLastError();
}

}  // namespace sc

#ifdef SC_BLEND_STATS
extern "C" __attribute__((visibility("default"))) int sc_debug_blend_stats(unsigned long long *host, int64_t n_tiles,
                                                                            int reset)
{
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, sc::g_blend_dbg) != cudaSuccess) return 2;
    if (reset) return cudaMemset(p, 0, sizeof(sc::g_blend_dbg)) == cudaSuccess ? 0 : 2;
    const size_t bytes = sizeof(unsigned long long) * 8 * (size_t)std::min<int64_t>(n_tiles, sc::kDbgTiles);
    return cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif
