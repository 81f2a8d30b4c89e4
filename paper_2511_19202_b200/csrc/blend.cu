// Stage (e): per-tile front-to-back alpha blending.
//
// Reference: composite_tiles (sc/_kernels.py:190-275) + finish()
// (sc/raster.py:267-282).  One CTA per 16x16 tile, one thread per pixel,
// each warp owning an 8x4 pixel block (lane = 8 * row + col).
//
// Entries are staged through shared memory in batches of 256, double
// buffered: the records of batch i+1 are gathered into registers while
// batch i is blended, so the HBM/L2 gather latency hides behind the math.
// Each warp then ballots the batch 32 entries at a time: an entry is walked
// only if its exact f64 pixel window (sc_splat.win, from the projection)
// intersects the warp's ALIVE pixels (32-bit mask vs the window's 8x4
// footprint), so saturated pixels cost nothing even while a silhouette pixel
// of the same warp keeps the warp busy.  Pixels retire after compositing
// once T < stop_transmittance (A8 step 7); warps stop when all 32 retired
// and the CTA stops when every warp has.  fp32 arithmetic (tolerance stated
// in tests/test_gpu_parity.py).
#include <algorithm>

#include "common.cuh"

namespace sc {

constexpr int kBatch = kBlendThreads;

#ifdef SC_BLEND_STATS
// instrumented build only (libsplatcull_b200_dbg.so): per tile
// [entries, batches walked, (entry, warp) hits, pixel evaluations, cycles, 0, 0, 0]
constexpr int kDbgTiles = 32400;
__device__ unsigned long long g_blend_dbg[kDbgTiles * 8];
#endif

struct __align__(16) BlendBuf {
    float4 geo[kBatch];   // mx, my, 0.5 a, b
    float4 pho[kBatch];   // 0.5 c, opacity, p_min, r
    float2 gb[kBatch];    // g, b
    short4 win[kBatch];   // x0, x1, y0, y1 (inclusive, absolute pixels)
    uint32_t idx[kBatch];
};

// 32-bit footprint of window w on the 8x4 block at (bx0, by0)
__device__ __forceinline__ uint32_t block_mask(short4 w, int bx0, int by0)
{
    const int lo = max((int)w.x, bx0), hi = min((int)w.y, bx0 + 7);
    const int rlo = max((int)w.z, by0), rhi = min((int)w.w, by0 + 3);
    if (lo > hi || rlo > rhi) return 0u;
    const uint32_t cols = (0xFFu >> (7 - (hi - bx0))) & (0xFFu << (lo - bx0));
    const uint32_t rows = (0x01010101u << (8 * (rlo - by0))) & (0x01010101u >> (8 * (3 - (rhi - by0))));
    return cols * rows;
}

__global__ void __launch_bounds__(kBlendThreads) k_blend(const sc_splat *__restrict__ splats, int64_t n_splats,
                                                         const uint32_t *__restrict__ entry_idx,
                                                         const uint32_t *__restrict__ tile_off, int width, int height,
                                                         int n_tx, float stop_t, float bg_r, float bg_g, float bg_b,
                                                         int record, float *image, float *trans, float *csum,
                                                         float *cmax)
{
    __shared__ BlendBuf sb[2];
    const int tile = blockIdx.x;
    const int tyi = tile / n_tx, txi = tile - tyi * n_tx;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int bx0 = txi * kTile + (wid & 1) * 8, by0 = tyi * kTile + (wid >> 1) * 4;
    const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
    const bool inside = px < width && py < height;
    const float fpx = (float)px, fpy = (float)py;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, cs = 0.0f;
    bool done = !inside;
    bool warp_done = __all_sync(0xffffffffu, done);
    const uint32_t start = tile_off[tile], end = tile_off[tile + 1];

    // register staging of one batch (this thread's entry)
    float4 ra = make_float4(0.f, 0.f, 0.f, 0.f), rb = ra, rc = ra;
    uint32_t rs = 0;
    bool rv = false;
    auto fetch = [&](uint32_t base) {
        const uint32_t e = base + tid;
        rv = e < end;
        if (rv) {
            uint32_t s = __ldg(entry_idx + e);
            if ((int64_t)s >= n_splats) s = 0;   // only reachable on workspace overflow
            const float4 *src = reinterpret_cast<const float4 *>(splats + s);
            ra = __ldg(src);
            rb = __ldg(src + 1);
            rc = __ldg(src + 2);
            rs = s;
        }
    };
    fetch(start);
    int buf = 0;
#ifdef SC_BLEND_STATS
    unsigned long long d_batches = 0, d_hits = 0, d_evals = 0;
    const long long d_t0 = clock64();
#endif
    for (uint32_t base = start; base < end; base += kBatch) {
#ifdef SC_BLEND_STATS
        d_batches++;
#endif
        BlendBuf &B = sb[buf];
        B.geo[tid] = ra;
        B.pho[tid] = rb;
        B.gb[tid] = make_float2(rc.x, rc.y);
        if (rv) {
            const uint32_t w01 = __float_as_uint(rc.z), w23 = __float_as_uint(rc.w);
            B.win[tid] = make_short4((short)(w01 & 0xFFFF), (short)(w01 >> 16), (short)(w23 & 0xFFFF),
                                     (short)(w23 >> 16));
        } else {
            B.win[tid] = make_short4(1, 0, 1, 0);
        }
        B.idx[tid] = rs;
        if (__syncthreads_and(warp_done)) break;
        if (base + kBatch < end) fetch(base + kBatch);   // overlaps the blending below
        const int nb = (int)min((uint32_t)kBatch, end - base);
        if (!warp_done) {
            for (int k0 = 0; k0 < nb; k0 += 32) {
                const uint32_t alive = __ballot_sync(0xffffffffu, !done);
                const int jj = k0 + lane;
                const bool hit = jj < nb && (block_mask(B.win[jj], bx0, by0) & alive) != 0u;
                uint32_t m = __ballot_sync(0xffffffffu, hit);
                while (m) {
                    const int j = k0 + __ffs(m) - 1;
                    m &= m - 1;
                    const short4 w = B.win[j];
                    float contrib = 0.0f;
#ifdef SC_BLEND_STATS
                    d_hits += (lane == 0);
                    d_evals += (!done && px >= w.x && px <= w.y && py >= w.z && py <= w.w);
#endif
                    if (!done && px >= w.x && px <= w.y && py >= w.z && py <= w.w) {
                        const float4 g = B.geo[j];
                        const float4 p = B.pho[j];
                        const float dx = fpx - g.x, dy = fpy - g.y;
                        const float power = -(g.z * dx * dx + p.x * dy * dy) - g.w * dx * dy;
                        if (!(power > 0.0f || power < p.z)) {
                            const float alpha = fminf(0.99f, p.y * __expf(power));
                            const float2 c2 = B.gb[j];
                            contrib = alpha * T;
                            cr += contrib * p.w;
                            cg += contrib * c2.x;
                            cb += contrib * c2.y;
                            T = T * (1.0f - alpha);
                            if (T < stop_t) done = true;
                        }
                    }
                    if (record) {
                        cs += contrib;
                        float mxc = contrib;
                        for (int o = 16; o > 0; o >>= 1) mxc = fmaxf(mxc, __shfl_xor_sync(0xffffffffu, mxc, o));
                        if (lane == 0 && mxc > 0.0f)
                            atomicMax(reinterpret_cast<int *>(cmax) + B.idx[j], __float_as_int(mxc));
                    }
                }
                warp_done = __all_sync(0xffffffffu, done);
                if (warp_done) break;
            }
        }
        buf ^= 1;
    }
#ifdef SC_BLEND_STATS
    for (int o = 16; o > 0; o >>= 1) {
        d_hits += __shfl_down_sync(0xffffffffu, d_hits, o);
        d_evals += __shfl_down_sync(0xffffffffu, d_evals, o);
    }
    if (tile < kDbgTiles) {
        unsigned long long *dd = g_blend_dbg + 8 * (size_t)tile;
        if (lane == 0) {
            atomicAdd(dd + 2, d_hits);
            atomicAdd(dd + 3, d_evals);
        }
        if (tid == 0) {
            dd[0] = end - start;
            dd[1] = d_batches;
            dd[4] = (unsigned long long)(clock64() - d_t0);
        }
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
                         const sc_camera &cam, const sc_opts &opts, const sc_frame_out &out, int64_t n_splats,
                         cudaStream_t st)
{
    const int n_tx = (cam.width + kTile - 1) / kTile, n_ty = (cam.height + kTile - 1) / kTile;
    SC_LAUNCH(k_blend, n_tx * n_ty, kBlendThreads, 0, st, splats, n_splats, entry_idx, tile_off, cam.width,
              cam.height, n_tx, (float)opts.stop_transmittance, (float)opts.background[0],
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
    const size_t bytes = sizeof(unsigned long long) * 8 * (size_t)std::min<int64_t>(n_tiles, sc::kDbgTiles);
    if (reset) return (int)cudaMemset(sc::g_blend_dbg, 0, sizeof(sc::g_blend_dbg)) == 0 ? 0 : 2;
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, sc::g_blend_dbg) != cudaSuccess) return 2;
    return cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif
