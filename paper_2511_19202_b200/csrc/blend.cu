// Stage (e): per-tile front-to-back alpha blending.
//
// Reference: composite_tiles (sc/_kernels.py:190-275) + finish()
// (sc/raster.py:267-282).  One CTA per 16x16 tile, one thread per pixel,
// each warp owning an 8x4 pixel block.  Splat records of the tile's entries
// are staged through shared memory in batches of 256 (one coalesced 48-byte
// record per thread); each warp then ballots the batch against its pixel
// block so it only walks the entries whose exact f64 pixel window
// (sc_splat.win, computed by the projection) touches it.  Pixels retire
// after compositing once T < stop_transmittance (A8 step 7), warps stop when
// all 32 pixels retired and the CTA stops loading batches when every warp
// has.  Arithmetic is fp32 (tolerance stated in tests/test_gpu_parity.py).
#include <algorithm>

#include "common.cuh"

namespace sc {

constexpr int kBatch = 256;

struct __align__(16) BlendBatch {
    float mx[kBatch], my[kBatch];
    float ha[kBatch], b[kBatch], hc[kBatch];
    float op[kBatch], pmin[kBatch];
    float r[kBatch], g[kBatch], bl[kBatch];
    short4 win[kBatch];
    uint32_t idx[kBatch];
};

__global__ void __launch_bounds__(kBlendThreads) k_blend(const sc_splat *__restrict__ splats, int64_t n_splats,
                                                         const uint32_t *__restrict__ entry_idx,
                                                         const uint32_t *__restrict__ tile_off, int width, int height,
                                                         int n_tx, float stop_t, float bg_r, float bg_g, float bg_b,
                                                         int record, float *image, float *trans, float *csum,
                                                         float *cmax)
{
    __shared__ BlendBatch sb;
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

    for (uint32_t base = start; base < end; base += kBatch) {
        if (__syncthreads_and(warp_done)) break;
        const uint32_t e = base + tid;
        if (e < end) {
            uint32_t s = entry_idx[e];
            if ((int64_t)s >= n_splats) s = 0;   // only reachable on workspace overflow
            const float4 *src = reinterpret_cast<const float4 *>(splats + s);
            const float4 a = __ldg(src), c = __ldg(src + 1), d = __ldg(src + 2);
            sb.mx[tid] = a.x;
            sb.my[tid] = a.y;
            sb.ha[tid] = a.z;
            sb.b[tid] = a.w;
            sb.hc[tid] = c.x;
            sb.op[tid] = c.y;
            sb.pmin[tid] = c.z;
            sb.r[tid] = c.w;
            sb.g[tid] = d.x;
            sb.bl[tid] = d.y;
            const uint32_t w01 = __float_as_uint(d.z), w23 = __float_as_uint(d.w);
            sb.win[tid] = make_short4((short)(w01 & 0xFFFF), (short)(w01 >> 16), (short)(w23 & 0xFFFF),
                                      (short)(w23 >> 16));
            sb.idx[tid] = s;
        } else {
            sb.win[tid] = make_short4(1, 0, 1, 0);
        }
        __syncthreads();
        const int nb = (int)std::min<uint32_t>(kBatch, end - base);
        if (!warp_done) {
            for (int k0 = 0; k0 < nb; k0 += 32) {
                const int jj = k0 + lane;
                bool hit = false;
                if (jj < nb) {
                    const short4 w = sb.win[jj];
                    hit = w.x <= bx0 + 7 && w.y >= bx0 && w.z <= by0 + 3 && w.w >= by0;
                }
                uint32_t m = __ballot_sync(0xffffffffu, hit);
                while (m) {
                    const int j = k0 + __ffs(m) - 1;
                    m &= m - 1;
                    const short4 w = sb.win[j];
                    float contrib = 0.0f;
                    if (!done && px >= w.x && px <= w.y && py >= w.z && py <= w.w) {
                        const float dx = fpx - sb.mx[j], dy = fpy - sb.my[j];
                        const float power = -(sb.ha[j] * dx * dx + sb.hc[j] * dy * dy) - sb.b[j] * dx * dy;
                        if (!(power > 0.0f || power < sb.pmin[j])) {
                            const float alpha = fminf(0.99f, sb.op[j] * __expf(power));
                            contrib = alpha * T;
                            cr += contrib * sb.r[j];
                            cg += contrib * sb.g[j];
                            cb += contrib * sb.bl[j];
                            T = T * (1.0f - alpha);
                            if (T < stop_t) done = true;
                        }
                    }
                    if (record) {
                        cs += contrib;
                        float mxc = contrib;
                        for (int o = 16; o > 0; o >>= 1) mxc = fmaxf(mxc, __shfl_xor_sync(0xffffffffu, mxc, o));
                        if (lane == 0 && mxc > 0.0f)
                            atomicMax(reinterpret_cast<int *>(cmax) + sb.idx[j], __float_as_int(mxc));
                    }
                }
                warp_done = __all_sync(0xffffffffu, done);
                if (warp_done) break;
            }
        }
        __syncthreads();
    }
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
