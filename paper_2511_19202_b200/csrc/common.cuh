// Shared device helpers and internal layouts for libsplatcull_b200.so (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "splatcull_b200.h"

namespace sc {

constexpr int kTile = 16;              // blend CTA tile edge (frame path; 8 warps of 8x4 pixel blocks)
constexpr int kCullThreads = 128;      // one MLP row per thread (tcgen05 M = 128)
#ifndef SC_CULL_TILES
#define SC_CULL_TILES 8
#endif
constexpr int kCullTilesPerChunk = SC_CULL_TILES;  // chunk = 1024 (instance, gaussian) pairs
constexpr int kChunk = kCullThreads * kCullTilesPerChunk;
constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = 4096;                          // radix sort tile (count matrix sizing)
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kBlendThreads = 256;

// Per-frame, per-instance state written by the prep kernel.
struct InstFrame {
    double corr;          // (f_train / focal) / s   (Eq. 2)
    float fwd_local[3];   // R^T camera forward
    int32_t visible;      // survived the bounding-sphere cull
    uint32_t chunk_begin; // exclusive prefix of chunk counts
    uint32_t n_chunks;
    // MLP inputs in the instance frame (f32): R^T (m' - c) = s m + cam_local
    float cam_local[3];   // R^T (t - c)
    float s;              // uniform instance scale
    float dn_a, dn_b;     // normalised distance = clamp(d_r dn_a + dn_b, -1, 1)
    int32_t inside;       // sphere strictly inside the frustum: every pair passes the per-pair test
    int32_t gate;         // 1: every pair is queried (d_t >= d_near), 0: none, -1: per-pair f64 test
};

// Screen band of a render in pixel rows [y0, y1) and tile rows [t0, t1) of
// `ts`-pixel tiles (sc_opts.band_*; the whole image [0, ts n_ty) when
// band_y1 <= 0).  Bands need tile_size 16 (api.cu check_opts), so the band's
// tile rows are also blend-CTA rows.
struct Band {
    int y0, y1, t0, t1;
};
__host__ __device__ __forceinline__ Band band_of(const sc_opts &o, int height, int ts)
{
    const int n_ty = (height + ts - 1) / ts;
    Band b{0, n_ty * ts, 0, n_ty};
    if (o.band_y1 > 0) {
        b.t0 = o.band_y0 / ts;
        b.t1 = (o.band_y1 + ts - 1) / ts;
        b.t1 = b.t1 < n_ty ? b.t1 : n_ty;
        b.y0 = b.t0 * ts;
        b.y1 = b.t1 * ts;
    }
    return b;
}

// Margin-mode frustum pad in pixels (B3, oracle/sc_oracle.c:margin_pad): the
// projected radius is ceil(3 sqrt(lambda)) with lambda <= (3 sigma f G / tz)^2
// / 9 + dilation, so radius <= 3 sigma (f / tz) G + 3 sqrt(dilation) + 1;
// at the default dilation 0.3 the pad is 3 px.  IEEE sqrt: identical on host
// and device.
__host__ __device__ __forceinline__ double margin_pad(double dilation)
{
    const double p = 3.0 * sqrt(dilation > 0.0 ? dilation : 0.0) + 1.0 + 1e-6;
    return p > 3.0 ? p : 3.0;
}

// Internal counters block (device), zeroed per frame together with the stats.
struct Counters {
    unsigned long long chunk_ticket;   // dynamic chunk assignment for the cull kernel
    unsigned long long total_chunks;
    unsigned long long survivors;      // = stats.survivors (u64 copy for kernels)
    unsigned long long passed;
    unsigned long long entries;
    unsigned long long entries_eff;    // entries, or 0 when they overflow the workspace
    unsigned long long dmin_inv;       // ~bits(min passed depth)  (atomicMax of ~bits; 0 = none)
    unsigned long long dmax;           // bits(max passed depth)   (positive doubles order as u64)
    unsigned long long tie_runs;       // runs of equal depth keys found by the tie-fix
    unsigned long long tie_long;       // ... of which longer than 8 (one CTA each)
    unsigned long long proj_deferred;  // splats the f32 projection left to the exact kernel
    double key_dmin, key_scale;        // frame path: depth-key quantisation from the instance spheres (k_prep)
    // dynamic tile tickets of the radix up/downsweeps (zero between launches: the last
    // CTA to finish resets them), so a sweep sharing the GPU with another stream's
    // kernels does not wait on CTAs that are not resident yet
    unsigned long long rs_next, rs_done;
    unsigned long long rs_scan_n;      // radix pass: 256 x this frame's tiles (the count matrix's length)
    unsigned long long blend_next;     // persistent blend warps: next short (tile, block) list of the LPT order
    unsigned long long blend_long_next;   // ... next long list (one CTA each)
    unsigned long long blend_n_long;      // ... number of long lists at the head of the order (k_tile_order)
    unsigned int order_hist[33];          // LPT buckets of the (tile, block) lists (k_order_hist)
    unsigned int order_cursor[33];        // ... slots handed out per bucket (k_order_scatter)
};

// Workspace carve-out (all offsets 256-byte aligned), see api.cu:carve().
struct Ws {
    InstFrame *inst;                 // [n_instances]
    unsigned long long *chunk_state; // [max_chunks] (instance << 32) | chunk index within the instance
    uint32_t *chunk_cnt;             // [max_chunks] survivors per chunk -> exclusive offsets
    uint32_t *chunk_inst;            // [max_chunks] the instance owning each chunk (k_chunk_map)
    uint16_t *chunk_stage;           // [max_chunks][kChunk] survivors of each chunk (offset in the chunk)
    Counters *ctr;
    sc_survivor *surv;               // [capS]
    sc_splat *splats;                // [capS]
    sc_window *wins;                 // [capS]
    uint32_t *key_a, *key_b;         // [max(capS, 4096)]  depth keys (ping-pong); key_b also the deferred /
                                     // tie-run / emission-total lists
    uint2 *pv_a, *pv_b;              // [capS]  (survivor index, packed pixel window) riding the depth sort
    double *depth64;                 // [capS]  stage-level API only
    ushort4 *rect;                   // [capS]  tx0, tx1, ty0, ty1 (stage-level API only)
    uint32_t *ekey_a, *ekey_b;       // [capE]   (aliases: see api.cu layout())
    uint32_t *eval_a, *eval_b;       // [capE]
    uint32_t *tile_off;              // [n_tiles_ref + 1] stage API: reference tile offsets
    uint32_t *task_order;            // [8 n_tiles] blend dispatch order over (tile, block) lists (longest first)
    uint32_t *boff;                  // [8 n_tiles + 1] offsets of the per-(tile, 8x4 block) entry lists
    uint32_t *rs_counts;             // radix pass digit counts -> bases, digit-major [256][nblk_max]
    uint32_t *scan_part;             // scan partials
    int64_t capS, capE, max_chunks, nblk_max, n_tiles;   // n_tiles: 16x16 blend tiles (frame path)
    int n_tx, n_ty;
    int ts, n_tx_ref;                // reference tile size (sc_opts.tile_size) and its tile columns
    int64_t n_tiles_ref;             // reference tiles (stage API binning)
};

// ------------------------------------------------------------------------
// float64 helpers.  TUs that include the bit-exact f64 paths are compiled
// with -fmad=false, so plain operators give unfused IEEE mul/add exactly as
// the reference's numba kernels (fastmath=False, no contraction).
// ------------------------------------------------------------------------

// B2 instancing: mean' = s (R m) + t in f64, rounded to f32 (Asset dtype).
__device__ __forceinline__ float3 inst_mean(const sc_instance_rec &in, float mx, float my, float mz)
{
    double m0 = mx, m1 = my, m2 = mz;
    double v0 = in.R[0] * m0 + in.R[1] * m1 + in.R[2] * m2;
    double v1 = in.R[3] * m0 + in.R[4] * m1 + in.R[5] * m2;
    double v2 = in.R[6] * m0 + in.R[7] * m1 + in.R[8] * m2;
    return make_float3(__double2float_rn(in.s * v0 + in.t[0]), __double2float_rn(in.s * v1 + in.t[1]),
                       __double2float_rn(in.s * v2 + in.t[2]));
}

// q' = q_i (x) q (Hamilton product, wxyz), f64 -> f32.
__device__ __forceinline__ float4 inst_quat(const sc_instance_rec &in, float4 q)
{
    double w1 = in.q[0], x1 = in.q[1], y1 = in.q[2], z1 = in.q[3];
    double w2 = q.x, x2 = q.y, y2 = q.z, z2 = q.w;
    return make_float4(__double2float_rn(w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2),
                       __double2float_rn(w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2),
                       __double2float_rn(w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2),
                       __double2float_rn(w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2));
}

// camera-space position of a world point, same association as the reference
// projection (sc/_kernels.py:35-43)
__device__ __forceinline__ void cam_xyz(const sc_camera &c, double m0, double m1, double m2, double &tx,
                                        double &ty, double &tz)
{
    const double *R = c.rot;
    tx = R[0] * (m0 - c.pos[0]) + R[1] * (m1 - c.pos[1]) + R[2] * (m2 - c.pos[2]);
    ty = R[3] * (m0 - c.pos[0]) + R[4] * (m1 - c.pos[1]) + R[5] * (m2 - c.pos[2]);
    tz = R[6] * (m0 - c.pos[0]) + R[7] * (m1 - c.pos[1]) + R[8] * (m2 - c.pos[2]);
}

// Packed pixel window (frame path sort payload): the window clamped to the
// image, x0 | y0 << 12 | (x1 - x0) << 24 | (y1 - y0) << 28 when it is at most
// 16 x 16 pixels and y0 < 4095; else kWinEscape (read sc_window from the
// array) or kWinEmpty.  Both sentinels have y0 = 4095, never a compact value.
constexpr uint32_t kWinEmpty = 0xFFFFFFFFu;
constexpr uint32_t kWinEscape = 0xFFFFFFFEu;

__host__ __device__ __forceinline__ uint32_t pack_window(int x0, int x1, int y0, int y1, int width, int height)
{
    x0 = x0 > 0 ? x0 : 0;
    y0 = y0 > 0 ? y0 : 0;
    x1 = x1 < width - 1 ? x1 : width - 1;
    y1 = y1 < height - 1 ? y1 : height - 1;
    if (x0 > x1 || y0 > y1) return kWinEmpty;
    if (x1 - x0 > 15 || y1 - y0 > 15 || x0 > 4095 || y0 >= 4095) return kWinEscape;
    return (uint32_t)x0 | ((uint32_t)y0 << 12) | ((uint32_t)(x1 - x0) << 24) | ((uint32_t)(y1 - y0) << 28);
}

// -> false for an empty window
__device__ __forceinline__ bool unpack_window(uint32_t p, uint32_t idx, const sc_window *wins, int width, int height,
                                              int &x0, int &x1, int &y0, int &y1)
{
    if (p == kWinEmpty) return false;
    if (p == kWinEscape) {
        const uint2 w = __ldg(reinterpret_cast<const uint2 *>(wins + idx));
        x0 = max((int)(int16_t)(w.x & 0xFFFF), 0);
        x1 = min((int)(int16_t)(w.x >> 16), width - 1);
        y0 = max((int)(int16_t)(w.y & 0xFFFF), 0);
        y1 = min((int)(int16_t)(w.y >> 16), height - 1);
        return x0 <= x1 && y0 <= y1;
    }
    x0 = (int)(p & 0xFFFu);
    y0 = (int)((p >> 12) & 0xFFFu);
    x1 = x0 + (int)((p >> 24) & 0xFu);
    y1 = y0 + (int)(p >> 28);
    return true;
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// order-preserving float -> uint32 radix key
__device__ __forceinline__ uint32_t float_key(float f)
{
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

}  // namespace sc

// launch bookkeeping (api.cu)
extern "C" void sc_note_launch(void);
#define SC_LAUNCH(kernel, grid, block, smem, stream, ...)                                    \
    do {                                                                                      \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                           \
        sc_note_launch();                                                                     \
    } while (0)

// internal launchers (host)
namespace sc {
// SM count of the current device (cached per device)
int sm_count();
// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the current device,
// set once per device (the attribute is per device context)
cudaError_t smem_attr_once(const void *func, int bytes);
cudaError_t launch_prep(const sc_scene &scene, const sc_camera &cam, const sc_opts &opts, const Ws &ws,
                        sc_frame_stats *stats, cudaStream_t st);
cudaError_t launch_cull(const sc_scene &scene, const sc_camera &cam, const sc_opts &opts, const Ws &ws,
                        sc_survivor *out, int64_t cap, sc_frame_stats *stats, cudaStream_t st);
// exclusive scan of uint32 (n from device or host); total -> *total_out (u64) / *stat_out (i64)
cudaError_t scan_excl(const uint32_t *in, uint32_t *out, const unsigned long long *n_dev, int64_t n_max,
                      uint32_t *part, unsigned long long *total_out, int64_t *stat_out, cudaStream_t st);
cudaError_t launch_project(const sc_scene &scene, const sc_survivor *surv, const unsigned long long *n_dev,
                           int64_t n_max, const sc_camera &cam, const sc_opts &opts, sc_splat *splats,
                           sc_window *wins, double *depth64, ushort4 *rect, uint32_t *keys, uint2 *pv,
                           double *dbg_f64, int32_t *dbg_rect, uint8_t *dbg_flags, sc_frame_stats *stats,
                           Counters *ctr, uint32_t *defer_list, cudaStream_t st);
// equal depth keys -> (f64 depth, survivor index) order; depth from depth64 or
// recomputed from the survivor (project.cu, -fmad=false)
// scratch: n_max doubles, free during the tie-fix (long runs sort their f64 depths there)
cudaError_t launch_tiefix(const sc_scene &scene, const sc_survivor *surv, const sc_camera &cam, const uint32_t *keys,
                          uint2 *pv, const double *depth64, const unsigned long long *n_dev, int64_t n_max,
                          uint32_t *run_list, double *scratch, Counters *ctr, sc_frame_stats *stats, cudaStream_t st);
cudaError_t launch_bin(const Ws &ws, const sc_scene &scene, const sc_survivor *surv, const unsigned long long *n_dev,
                       int64_t n_max, const sc_camera &cam, const sc_window *wins, sc_frame_stats *stats, bool blocks,
                       uint32_t **order_out, uint32_t **entries_out, uint32_t **keys_out, uint32_t *dbg_order,
                       cudaStream_t st);
// Blend input, one of:
//  * block lists (frame path): boff [8 n_tiles + 1], vals = survivor per entry,
//    keys = block id << 10 | block-relative window;
//  * tile lists (stage-level API): tile_off [n_tiles + 1], vals = entry_idx,
//    keys = NULL (windows read from the splat records).
struct BlendLists {
    const uint32_t *offsets;
    const uint32_t *vals;
    const uint32_t *keys;
    const sc_window *wins;   // tile lists only: windows to clip per warp block
    bool blocks;
    Counters *ctr;   // block lists: the frame's counters (blend tickets, list order; zeroed per frame), else NULL
};
cudaError_t launch_blend(const sc_splat *splats, const BlendLists &lists, const sc_camera &cam, const sc_opts &opts,
                         const sc_frame_out &out, int64_t n_splats, uint32_t *task_order, cudaStream_t st);
cudaError_t launch_vis_mlp(const sc_vis_weights *w, const float *x, int64_t n, float *logits,
                           cudaStream_t st);
cudaError_t launch_encode_features(const float *params, const float *x, int64_t n, uint16_t *feat,
                                   cudaStream_t st);
}  // namespace sc
