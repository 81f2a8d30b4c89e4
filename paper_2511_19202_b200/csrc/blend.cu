// Stage (e): per-tile front-to-back alpha blending.
//
// Reference: composite_tiles (sc/_kernels.py:190-275) + finish()
// (sc/raster.py:267-282).  Semantics per pixel are the reference's: walk the
// tile's entries in (depth, index) order, skip splats with alpha0 < 1/255,
// composite inside the splat's pixel window when p_min <= power <= 0,
// alpha = min(0.99, alpha0 e^power), retire the pixel after compositing once
// T < stop_transmittance.  fp32 arithmetic (tolerance stated in
// tests/test_gpu_parity.py).
//
// B200 mapping — one CTA per 16x16 tile, 8 warps, no CTA barrier at all:
//   * a warp owns an 8x4 pixel block (lane = 8 row + col) and walks its own
//     depth-ordered (tile, block) list; CTAs are dispatched heaviest tile first
//     (LPT order by log2 entry count, k_tile_order);
//   * meta stream: the list's (index, window code) pairs are read 128 entries per
//     step (4 per lane, one step prefetched in registers); entries whose
//     footprint misses every still-alive pixel are dropped on the spot, the
//     others are compacted, in order, into a per-warp hit queue in shared memory
//     (alive only shrinks, so the mask at queue time is a superset: exact);
//   * record pipeline: 32 queued hits at a time become a stage whose 32-byte
//     splat records are cp.async'd into one of 4 shared slots; up to 3 stages
//     are in flight while the oldest is blended;
//   * blending a stage: the warp transposes the 32 footprints (32x32 bit
//     transpose over shuffles) so each lane walks only the entries covering its
//     own pixel; the warp iterates max-over-lanes times;
//   * a warp exits when its 32 pixels have retired.
// History (ncu, config-3 far view): a 256-entry CTA batch behind a barrier was
// barrier-stall bound (42 ms); barrier-free warps with per-hit shuffles were
// then bound by re-gathering windows (65 GB DRAM per launch), by the
// dependent-load chain per 32 entries (-> cp.async pipeline), by tile lists
// (-> per-block lists) and by streaming entries that touch only retired pixels
// (-> hit compaction: in the heaviest tiles ~80 % of entries miss every alive
// pixel because a few pixels never saturate).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace sc {

#ifdef SC_BLEND_STATS
// instrumented build only (libsplatcull_b200_dbg.so): per tile
// [entries, 32-entry slots walked, (entry, warp) hits, pixel evaluations, max warp cycles, warp iterations, 0, 0]
constexpr int kDbgTiles = 32400;
__device__ unsigned long long g_blend_dbg[kDbgTiles * 8];
// per (tile, block) list of the frame path: [entries, entries streamed before the walk stopped]
__device__ unsigned int g_blend_used[kDbgTiles * 8 * 2];
#endif

#ifndef SC_BLEND_WARPS
#define SC_BLEND_WARPS 4
#endif
// warps per CTA: 4 (a CTA walk splits each 32-hit x 4 chunk over 4 warps; 8 warps spent 18 % of
// their stall samples at the chunk barriers waiting for the slowest segment: blend -18 %; 2 warps
// leave the long lists too few warps)
constexpr int kBlendWarps = SC_BLEND_WARPS;
constexpr int kG = 32;                   // hits per record stage
constexpr int kStep = 128;               // meta entries per stream step (4 per lane)
constexpr int kHQ = 256;                 // hit queue capacity (>= kG + kStep)
#ifndef SC_BLEND_STAGES
#define SC_BLEND_STAGES 3
#endif
constexpr int kRecStages = SC_BLEND_STAGES;   // record stages: up to kRecStages - 1 in flight while the oldest
                                              // is blended (3: 5.9 KB per warp, 4 CTAs = 32 warps per SM)
#ifndef SC_HEAVY_PIXELS
#define SC_HEAVY_PIXELS 8
#endif
#ifndef SC_HEAVY_HITS
#define SC_HEAVY_HITS 8
#endif
constexpr int kMaxHeavyPixels = SC_HEAVY_PIXELS;   // ... and at most this many such pixels in the stage
constexpr int kHeavyHits = SC_HEAVY_HITS;          // a pixel covered by >= this many entries of a stage: entry-parallel
constexpr size_t kHQBytesW = sizeof(uint2) * kHQ;
constexpr size_t kStageMetaBytesW = sizeof(uint2) * kG * kRecStages;
constexpr size_t kRecBytesW = sizeof(float4) * 2 * kG * kRecStages;   // 32-byte sc_splat records
constexpr size_t kWarpSmem = kHQBytesW + kStageMetaBytesW + kRecBytesW;   // one warp's queues

// 32-bit footprint (lane = 8 row + col) of a block-relative window code
// x0 | x1 << 3 | y0 << 6 | y1 << 8 on the 8x4 block; 0 when x0 > x1
__device__ __forceinline__ uint32_t code_mask(uint32_t c)
{
    const uint32_t x0 = c & 7u, x1 = (c >> 3) & 7u, y0 = (c >> 6) & 3u, y1 = (c >> 8) & 3u;
    const uint32_t cols = (0xFFu >> (7u - x1)) & (0xFFu << x0) & 0xFFu;
    const uint32_t rows = (0x01010101u << (8u * y0)) & (0x01010101u >> (8u * (3u - y1)));
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

// e^x for x in [0, ln 255 + 1] (power - p_min once the window test passed): the same
// ex2.approx as __expf, without its denormal-result range fix-up (never taken here)
__device__ __forceinline__ float exp_nonneg(float x)
{
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x * 1.4426950408889634f));
    return r;
}

__device__ __forceinline__ int lo16(uint32_t w) { return (int)(int16_t)(w & 0xFFFFu); }
__device__ __forceinline__ int hi16(uint32_t w) { return (int)(int16_t)(w >> 16); }

__device__ __forceinline__ uint32_t smem_u32p(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32p(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32p(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// wait until at most n (0..3) cp.async groups are pending
__device__ __forceinline__ void cp_async_wait_dyn(uint32_t n)
{
    switch (n) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    default: cp_async_wait<3>(); break;
    }
}

constexpr uint32_t kNoEntry = 0xFFFFFFFFu;
constexpr uint32_t kEmptyCode = 0x0007u;   // x0 = 7 > x1 = 0

// Per-warp constants of one list walk.
struct WalkCtx {
    const sc_splat *__restrict__ splats;
    int64_t n_splats;
    const uint32_t *__restrict__ vals;
    const uint32_t *__restrict__ keys;
    const sc_window *__restrict__ wins;
    int blocks;
    int gx0, gy0;       // warp block origin, absolute pixels
    int bx1, by1;       // last pixel column / row of the block inside its tile (tile lists)
    float fpx, fpy;     // this lane's pixel
    float stop_t;
    int record;
    float *cmax;
    uint2 *hq;          // warp-private hit queue [kHQ] (index, footprint)
    uint2 *stage;       // [kRecStages][32] (index, footprint) of each record stage
    float4 *recs;       // [kRecStages][32][2]
    int lane;
};

// Per-pixel compositing state (one pixel per lane).
struct PixAcc {
    float T, cr, cg, cb, cs;
    bool done;
};

#ifdef SC_BLEND_STATS
struct WalkStats { unsigned long long slots, hits, evals, iters, meta; };
#define SC_WS_PARAM , WalkStats &d
#define SC_WS_ARG , d
#else
#define SC_WS_PARAM
#define SC_WS_ARG
#endif

// Entry-parallel compositing of one pixel pl over a record stage (grp: lane j's
// entry at grp[2 j]; cov bit j: entry j covers pl; T_in: pl's transmittance before
// the stage).  Lane j evaluates entry j's alpha at the pixel (alphas do not depend
// on T), an in-order warp prefix product of (1 - alpha) gives T before every
// entry, the reference's retirement cut (first T < stop after a composite) is a
// ballot and the colour a warp sum.  Same terms as the serial walk, products in
// tree order (fp32 rounding only).  Warp-uniform results: colour sums and T_out.
__device__ __forceinline__ void pixel_entry_parallel(const WalkCtx &c, const float4 *grp, uint32_t cov, float T_in,
                                                     float qx, float qy, uint32_t sidx, float &sr, float &sg,
                                                     float &sb, float &sc, float &T_out)
{
    const int lane = c.lane;
    float alpha = 0.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    if ((cov >> lane) & 1u) {
        const float4 *r = grp + lane * 2;
        const float4 g = r[0];
        const float4 p = r[1];
        const float dx = qx - g.x, dy = qy - g.y;
        const float power = -(g.z * dx * dx + p.x * dy * dy) - g.w * dx * dy;
        if (!(power > 0.0f || power < p.y)) {
            alpha = fminf(0.99f, exp_nonneg(power - p.y) * (1.0f / 255.0f));
            const __half2 rg = *reinterpret_cast<const __half2 *>(&p.z);
            const __half2 bx = *reinterpret_cast<const __half2 *>(&p.w);
            cr = __low2float(rg);
            cg = __high2float(rg);
            cb = __low2float(bx);
        }
    }
    // inclusive prefix product of (1 - alpha) over lanes 0..j
    float incl = 1.0f - alpha;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl *= y;
    }
    float excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 1.0f;
    const float t_before = T_in * excl, t_after = T_in * incl;
    // composited: a valid entry reached before the pixel retired
    const bool comp = alpha > 0.0f && t_before >= c.stop_t;
    const float contrib = comp ? alpha * t_before : 0.0f;
    if (c.record && contrib > 0.0f) atomicMax(reinterpret_cast<int *>(c.cmax) + sidx, __float_as_int(contrib));
    sr = contrib * cr;
    sg = contrib * cg;
    sb = contrib * cb;
    sc = contrib;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffffu, sr, o);
        sg += __shfl_xor_sync(0xffffffffu, sg, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
        if (c.record) sc += __shfl_xor_sync(0xffffffffu, sc, o);   // the contribution sum is a record output
    }
    const uint32_t compm = __ballot_sync(0xffffffffu, comp);
    T_out = compm ? __shfl_sync(0xffffffffu, t_after, 31 - __clz(compm)) : T_in;
}

// Blend one record stage onto the lanes' pixels: lane j holds entry j's splat
// index sidx and footprint fp (already masked by the alive pixels), its record at
// grp[2 j].  The warp transposes the 32 footprints so each lane walks only the
// entries covering its own pixel (max-over-lanes iterations); pixels covered by
// >= kHeavyHits of the stage's entries (when at most kMaxHeavyPixels) go
// entry-parallel instead -- the serial per-pixel chain (~150-200 cycles per
// composite) was the tail of the heaviest lists.
__device__ __forceinline__ void blend_stage(const WalkCtx &c, const float4 *grp, uint32_t sidx_lane, uint32_t fp,
                                            PixAcc &a SC_WS_PARAM)
{
    const int lane = c.lane;
    const uint32_t covers = transpose32(fp, lane);   // bit j: entry of lane j covers my pixel
    uint32_t heavy = __ballot_sync(0xffffffffu, __popc(covers) >= kHeavyHits);
    // when many pixels are heavy the lane-per-pixel loop is already busy on every lane
    if (__popc(heavy) > kMaxHeavyPixels) heavy = 0u;
    uint32_t mine = ((heavy >> lane) & 1u) ? 0u : covers;
    while (__any_sync(0xffffffffu, mine != 0u)) {
        const bool act = mine != 0u;
        const int j = act ? __ffs(mine) - 1 : lane;
        mine &= mine - 1u;
        const uint32_t sidx = c.record ? __shfl_sync(0xffffffffu, sidx_lane, j) : 0u;
#ifdef SC_BLEND_STATS
        d.evals += act;
        d.iters += (lane == 0);
#endif
        if (act) {
            const float4 *r = grp + j * 2;
            const float4 g = r[0];   // mx, my, 0.5 a, b
            const float4 p = r[1];   // 0.5 c, p_min, rgb (fp16 x3)
            const float dx = c.fpx - g.x, dy = c.fpy - g.y;
            const float power = -(g.z * dx * dx + p.x * dy * dy) - g.w * dx * dy;
            if (!(power > 0.0f || power < p.y)) {
                // opacity * e^power == e^(power - p_min) / 255
                const float alpha = fminf(0.99f, exp_nonneg(power - p.y) * (1.0f / 255.0f));
                const float contrib = alpha * a.T;
                const __half2 rg = *reinterpret_cast<const __half2 *>(&p.z);
                const __half2 bx = *reinterpret_cast<const __half2 *>(&p.w);
                a.cr += contrib * __low2float(rg);
                a.cg += contrib * __high2float(rg);
                a.cb += contrib * __low2float(bx);
                a.T = a.T * (1.0f - alpha);
                if (c.record) {
                    a.cs += contrib;
                    if (contrib > 0.0f) atomicMax(reinterpret_cast<int *>(c.cmax) + sidx, __float_as_int(contrib));
                }
                if (a.T < c.stop_t) {
                    a.done = true;
                    mine = 0u;
                }
            }
        }
    }
    uint32_t hv = heavy;
    while (hv) {
        const int pl = __ffs(hv) - 1;
        hv &= hv - 1u;
        const uint32_t cov = __shfl_sync(0xffffffffu, covers, pl);
        const float T_in = __shfl_sync(0xffffffffu, a.T, pl);
        const float qx = __shfl_sync(0xffffffffu, c.fpx, pl), qy = __shfl_sync(0xffffffffu, c.fpy, pl);
        float sr, sg, sb, sc, T_out;
        pixel_entry_parallel(c, grp, cov, T_in, qx, qy, sidx_lane, sr, sg, sb, sc, T_out);
        if (lane == pl) {
            a.cr += sr;
            a.cg += sg;
            a.cb += sb;
            a.cs += sc;
            a.T = T_out;
            if (T_out < c.stop_t) a.done = true;
        }
#ifdef SC_BLEND_STATS
        d.evals += __popc(cov) * (lane == pl);
        d.iters += (lane == 0);
#endif
    }
}

// Front-to-back compositing of entries [start, end) of the warp's stream onto
// the lanes that are not done (reference semantics, sc/_kernels.py:190-275).
__device__ __forceinline__ void walk_list(const WalkCtx &c, uint32_t start, uint32_t end, PixAcc &a SC_WS_PARAM)
{
    const int lane = c.lane;
#ifdef SC_BLEND_STATS
    d.meta = 0;
#endif
    if (__all_sync(0xffffffffu, a.done) || start >= end) return;
    const uint32_t lt = lanemask_lt();
    // meta of stream step [base, base + 128): entry base + 32 j + lane in (v[j], k[j])
    uint32_t va[4], ka[4], vb[4], kb[4];
    auto load_step = [&](uint32_t base, uint32_t *v, uint32_t *k) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t e = base + 32 * j + lane;
            v[j] = kNoEntry;
            k[j] = kEmptyCode;
            if (e < end) {
                v[j] = __ldg(c.vals + e);
                if (c.blocks) k[j] = __ldg(c.keys + e);   // block id << 10 | block-relative window
            }
        }
    };
    // footprint of an entry on this warp's block (tile lists: clip the record's window here)
    auto footprint = [&](uint32_t v, uint32_t k) -> uint32_t {
        if ((int64_t)v >= c.n_splats) return 0u;
        if (c.blocks) return code_mask(k & 0x3FFu);
        const uint2 w = __ldg(reinterpret_cast<const uint2 *>(c.wins + v));
        const int x0 = max(lo16(w.x), c.gx0), x1 = min(hi16(w.x), c.bx1);
        const int y0 = max(lo16(w.y), c.gy0), y1 = min(hi16(w.y), c.by1);
        if (x0 > x1 || y0 > y1) return 0u;
        return code_mask((uint32_t)((x0 - c.gx0) | ((x1 - c.gx0) << 3) | ((y0 - c.gy0) << 6) | ((y1 - c.gy0) << 8)));
    };

    uint32_t mbase = start;
    load_step(mbase, va, ka);
    if (mbase + kStep < end) load_step(mbase + kStep, vb, kb);
    bool meta_done = false;
    uint32_t hq_head = 0, hq_tail = 0;   // running counters (slot = counter % kHQ)
    uint32_t issued = 0, blended = 0;    // record stages
    for (;;) {
        const uint32_t alive = __ballot_sync(0xffffffffu, !a.done);
        if (!alive) break;
        // 1. stream meta until a full stage of hits is queued (or the list ends)
        while (!meta_done && hq_tail - hq_head < (uint32_t)kG) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t fp = footprint(va[j], ka[j]) & alive;
                const uint32_t bal = __ballot_sync(0xffffffffu, fp != 0u);
                if (fp) c.hq[(hq_tail + __popc(bal & lt)) & (kHQ - 1)] = make_uint2(va[j], fp);
                hq_tail += __popc(bal);
            }
            mbase += kStep;
            if (mbase >= end) {
                meta_done = true;
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    va[j] = vb[j];
                    ka[j] = kb[j];
                }
                if (mbase + kStep < end) load_step(mbase + kStep, vb, kb);
            }
        }
        __syncwarp();
        // 2. turn up to 32 queued hits into a record stage (cp.async of their records)
        const uint32_t queued = hq_tail - hq_head;
        const bool room = issued - blended < (uint32_t)kRecStages;
        if (room && (queued >= (uint32_t)kG || (meta_done && queued > 0))) {
            const uint32_t n = queued < (uint32_t)kG ? queued : (uint32_t)kG;
            const int slot = (int)(issued % kRecStages);
            uint2 h = make_uint2(kNoEntry, 0u);
            if ((uint32_t)lane < n) {
                h = c.hq[(hq_head + lane) & (kHQ - 1)];
                h.y &= alive;
            }
            c.stage[slot * kG + lane] = h;
            if (h.y) {
                const float4 *src = reinterpret_cast<const float4 *>(c.splats + h.x);
                float4 *dst = c.recs + (slot * kG + lane) * 2;
                cp_async16(dst, src);
                cp_async16(dst + 1, src + 1);
            }
            cp_async_commit();
            hq_head += n;
            issued++;
            // keep up to three stages in flight before blending the oldest
            if (issued - blended < (uint32_t)kRecStages && !(meta_done && hq_tail == hq_head)) continue;
        }
        if (issued == blended) {
            if (meta_done && hq_tail == hq_head) break;
            continue;
        }
        // 3. blend the oldest stage once its records have landed
        cp_async_wait_dyn(issued - blended - 1);
        __syncwarp();
        const int slot = (int)(blended % kRecStages);
        const uint2 m = c.stage[slot * kG + lane];
        const uint32_t alive_now = __ballot_sync(0xffffffffu, !a.done);
        const uint32_t fp = m.y & alive_now;
#ifdef SC_BLEND_STATS
        d.slots++;
        d.hits += __popc(__ballot_sync(0xffffffffu, fp != 0u)) * (lane == 0);
#endif
        if (__any_sync(0xffffffffu, fp != 0u)) blend_stage(c, c.recs + slot * kG * 2, m.x, fp, a SC_WS_ARG);
        __syncwarp();   // the slot is refilled by a later stage
        blended++;
    }
    cp_async_wait<0>();
    __syncwarp();
#ifdef SC_BLEND_STATS
    d.meta = min(mbase, end) - start;
#endif
}

// Frame path: one CTA per 16x16 tile, warp w = 8x4 block w, walking its own
// (tile, block) list.  Stage-level API (tile lists of ts x ts tiles): a tile is
// covered by ceil(ts / 8) x ceil(ts / 4) 8x4 blocks (the last ones clipped to
// the tile), 8 per CTA; every warp walks the whole tile list, clipping each
// record's window to its block.
template <int REC>
__global__ void __launch_bounds__(kBlendWarps * 32) k_blend(const sc_splat *__restrict__ splats, int64_t n_splats,
                                                      const uint32_t *__restrict__ offsets,
                                                      const uint32_t *__restrict__ vals,
                                                      const uint32_t *__restrict__ keys,
                                                      const sc_window *__restrict__ wins, int blocks,
                                                      const uint32_t *__restrict__ task_order, int tile_base,
                                                      int width, int height, int n_tx, int ts, int nbx, int nblk,
                                                      int ngroups, float stop_t, float bg_r, float bg_g, float bg_b,
                                                      float *image, float *trans, float *csum,
                                                      float *cmax)
{
    extern __shared__ float4 s_dyn[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WalkCtx c;
    c.splats = splats;
    c.n_splats = n_splats;
    c.vals = vals;
    c.keys = keys;
    c.wins = wins;
    c.blocks = blocks;
    c.stop_t = stop_t;
    c.record = REC;   // compile-time: the non-recording kernels carry no contribution code
    c.cmax = cmax;
    c.lane = lane;
    // this warp's private queues: hits [kHQ], stage metas [kRecStages][32], records [kRecStages][32][2]
    char *wbase = reinterpret_cast<char *>(s_dyn) + wid * kWarpSmem;
    c.hq = reinterpret_cast<uint2 *>(wbase);
    c.stage = reinterpret_cast<uint2 *>(wbase + kHQBytesW);
    c.recs = reinterpret_cast<float4 *>(wbase + kHQBytesW + kStageMetaBytesW);
#ifdef SC_BLEND_STATS
    WalkStats d{0, 0, 0, 0, 0};
    const long long d_t0 = clock64();
#endif
    const int cta = (int)blockIdx.x / ngroups;
    const int tile = (int)(task_order ? task_order[cta] : tile_base + cta);
    const int b = ((int)blockIdx.x - cta * ngroups) * kBlendWarps + wid;   // block within the tile
    if (b >= nblk) return;   // (no CTA barrier in this kernel)
    const int tyi = tile / n_tx, txi = tile - tyi * n_tx;
    const int byi = b / nbx, bxi = b - byi * nbx;
    c.gx0 = txi * ts + bxi * 8;
    c.gy0 = tyi * ts + byi * 4;
    c.bx1 = min(c.gx0 + 7, txi * ts + ts - 1);
    c.by1 = min(c.gy0 + 3, tyi * ts + ts - 1);
    const int px = c.gx0 + (lane & 7), py = c.gy0 + (lane >> 3);
    const bool inside = px <= c.bx1 && py <= c.by1 && px < width && py < height;
    c.fpx = (float)px;
    c.fpy = (float)py;
    PixAcc a{1.0f, 0.0f, 0.0f, 0.0f, 0.0f, !inside};
    // this warp's entry stream: its (tile, block) list in the frame path, else
    // the whole tile list (stage-level API; windows clipped from the records)
    const uint32_t start = blocks ? offsets[8 * tile + b] : offsets[tile];
    const uint32_t end = blocks ? offsets[8 * tile + b + 1] : offsets[tile + 1];
    walk_list(c, start, end, a SC_WS_ARG);
#ifdef SC_BLEND_STATS
    for (int o = 16; o > 0; o >>= 1) d.evals += __shfl_down_sync(0xffffffffu, d.evals, o);
    if (tile < kDbgTiles && lane == 0) {
        unsigned long long *dd = g_blend_dbg + 8 * (size_t)tile;
        atomicAdd(dd, (unsigned long long)(end - start));
        atomicAdd(dd + 1, d.slots);
        atomicAdd(dd + 2, d.hits);
        atomicAdd(dd + 3, d.evals);
        atomicMax(dd + 4, (unsigned long long)(clock64() - d_t0));
        atomicAdd(dd + 5, d.iters);
    }
#endif
    if (inside) {
        const int64_t p = (int64_t)py * width + px;
        image[3 * p + 0] = a.cr + a.T * bg_r;
        image[3 * p + 1] = a.cg + a.T * bg_g;
        image[3 * p + 2] = a.cb + a.T * bg_b;
        trans[p] = a.T;
        if (REC && csum) csum[p] = a.cs;
    }
}

// ---- long lists: one CTA per (tile, block) list (frame path) ----
//
// A few very long lists set the blend's tail (config-3 far view: 8.9K non-empty
// lists of mean 20K entries, the longest 137K; near view: one warp walking a
// 141K-entry list was the whole kernel's duration).  Lists of at least
// 2^SC_COOP_LOG2 entries are therefore walked by a whole CTA, exactly.
#ifndef SC_COOP_LOG2
#define SC_COOP_LOG2 10
#endif
constexpr int pow2_at_least(int x) { return x <= 1 ? 1 : 2 * pow2_at_least((x + 1) / 2); }
constexpr int kCoopQ = pow2_at_least(2 * kBlendWarps * kG + kBlendWarps * kStep);   // CTA hit queue (ring: 2 chunks + one stream step)
constexpr int kCoopChunk = kBlendWarps * kG;     // 256 hits per chunk, 32 per warp
constexpr int kCoopStep = kBlendWarps * kStep;   // 1024 meta entries per CTA stream step
struct CoopSmem {
    uint2 q[kCoopQ];                        // (splat index, footprint) of queued hits, list order
    uint2 stage[kBlendWarps][2][kG];        // per warp: the hits of its segment of the current / next chunk
    float4 recs[kBlendWarps][2][kG * 2];    // ... and their 32-byte splat records
    float4 seg[kBlendWarps][32];            // per segment, per pixel: (P, r, g, b) composited from T = 1
    float4 fin[32];                         // (T, r, g, b) of pixels retired by a segment re-composite
    uint32_t cnt[2][kBlendWarps];           // stream step: hits per warp (double-buffered by step parity)
    uint32_t ticket[2];
    uint32_t mask_x[64];                    // code_mask by table: column byte of (x0 | x1 << 3)
    uint32_t mask_y[16];                    // ... and row selector of (y0 | y1 << 2): mask = x * y
};
static_assert(sizeof(CoopSmem) <= kBlendWarps * kWarpSmem, "the CTA layout reuses the per-warp queues' bytes");
static_assert(kCoopQ >= 2 * kCoopChunk + kCoopStep, "queue holds two chunks plus one stream step");

// One list walked by the whole CTA.  The meta streams 1024 entries per step (128
// per warp) and hits (entries touching a still-alive pixel) are compacted in
// order into the CTA queue.  Each chunk of 256 queued hits is cut into 8
// consecutive segments of 32, one per warp; a warp composites its segment onto
// the alive pixels from T = 1 (blend_stage), giving per pixel the segment's
// transmittance product P_w and colour C_w.  After a barrier every warp combines
// the 8 segments in order (C += T C_w, T *= P_w) as long as T P_w >= stop: T is
// non-increasing along the list, so no pixel retired inside such a segment.  A
// pixel whose T would fall below stop inside segment w retires there: warp w
// re-composites that segment for it from its true T (pixel_entry_parallel: the
// reference's exact cut).  Alive shrinks chunk by chunk as in the serial walk, so
// entries behind retired pixels still never reach the queue.  Every CTA-level
// decision derives from state all warps hold identically (alive, counters).
// Accumulation order differs from the serial walk (fp32 rounding only).
__device__ void coop_list(const WalkCtx &c, CoopSmem &s, int wid, uint32_t start, uint32_t end, PixAcc &a,
                          bool &retired_here SC_WS_PARAM)
{
    const int lane = c.lane;
    const uint32_t lt = lanemask_lt();
    uint32_t va[4], ka[4], vb[4], kb[4];
    auto load_step = [&](uint32_t base, uint32_t *v, uint32_t *k) {   // this warp's 128 entries of a step
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t e = base + (uint32_t)(kStep * wid + 32 * j + lane);
            v[j] = kNoEntry;
            k[j] = kEmptyCode;
            if (e < end) {
                v[j] = __ldg(c.vals + e);
                k[j] = __ldg(c.keys + e);
            }
        }
    };
    uint32_t mbase = start;
    load_step(mbase, va, ka);
    if (mbase + kCoopStep < end) load_step(mbase + kCoopStep, vb, kb);
    bool meta_done = false;
    uint32_t qi = 0, qtail = 0;            // queue: next hit to issue, tail
    uint32_t issued = 0, blended = 0, step = 0;
    for (;;) {
        const uint32_t alive = __ballot_sync(0xffffffffu, !a.done);
        if (!alive) break;
        // 1. stream meta until two chunks are queued (or the list ends)
        while (!meta_done && qtail - qi < 2u * kCoopChunk) {
            uint32_t fp[4], bal[4], nw = 0;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                // (padding past the list end carries kEmptyCode: an empty mask)
                fp[j] = s.mask_x[ka[j] & 63u] * s.mask_y[(ka[j] >> 6) & 15u] & alive;
                bal[j] = __ballot_sync(0xffffffffu, fp[j] != 0u);
                nw += __popc(bal[j]);
            }
            if (lane == 0) s.cnt[step & 1][wid] = nw;
            __syncthreads();
            const uint32_t cw = lane < kBlendWarps ? s.cnt[step & 1][lane] : 0u;
            uint32_t off = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kBlendWarps; w++) {
                const uint32_t x = __shfl_sync(0xffffffffu, cw, w);
                off += w < wid ? x : 0u;
                tot += x;
            }
            uint32_t pos = qtail + off;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (fp[j]) s.q[(pos + __popc(bal[j] & lt)) & (kCoopQ - 1)] = make_uint2(va[j], fp[j]);
                pos += __popc(bal[j]);
            }
            qtail += tot;
            step++;
            mbase += kCoopStep;
            if (mbase >= end) {
                meta_done = true;
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    va[j] = vb[j];
                    ka[j] = kb[j];
                }
                if (mbase + kCoopStep < end) load_step(mbase + kCoopStep, vb, kb);
            }
        }
        __syncthreads();   // queued hits visible to every warp; the last chunk's seg / fin consumed
        // 2. record stages of the next chunks (one chunk in flight while one is blended)
        while (issued - blended < 2u) {
            const uint32_t avail = qtail - qi;
            if (avail == 0u || (!meta_done && avail < (uint32_t)kCoopChunk)) break;
            const uint32_t n = avail < (uint32_t)kCoopChunk ? avail : (uint32_t)kCoopChunk;
            const int slot = (int)(issued & 1u);
            const uint32_t k = 32u * (uint32_t)wid + (uint32_t)lane;
            uint2 h = make_uint2(kNoEntry, 0u);
            if (k < n) {
                h = s.q[(qi + k) & (kCoopQ - 1)];
                h.y &= alive;
            }
            s.stage[wid][slot][lane] = h;
            if (h.y) {
                const float4 *src = reinterpret_cast<const float4 *>(c.splats + h.x);
                float4 *dst = &s.recs[wid][slot][2 * lane];
                cp_async16(dst, src);
                cp_async16(dst + 1, src + 1);
            }
            cp_async_commit();
            qi += n;
            issued++;
        }
        if (issued == blended) break;   // the list is exhausted
        // 3. this warp's segment of the oldest chunk, composited from T = 1
        cp_async_wait_dyn(issued - blended - 1);
        __syncwarp();
        const int slot = (int)(blended & 1u);
        const uint2 m = s.stage[wid][slot][lane];
        const uint32_t fp = m.y & alive;
        PixAcc loc{1.0f, 0.0f, 0.0f, 0.0f, 0.0f, a.done};
        if (__any_sync(0xffffffffu, fp != 0u)) blend_stage(c, s.recs[wid][slot], m.x, fp, loc SC_WS_ARG);
        s.seg[wid][lane] = make_float4(loc.T, loc.cr, loc.cg, loc.cb);
        __syncthreads();
        // 4. combine the segments in list order (every warp, identical T and retirements; the
        // colour only in warp 0, which writes the pixels)
        int rw = -1;
        float tin = 0.0f;
        if (!a.done) {
#pragma unroll
            for (int w = 0; w < kBlendWarps; w++) {
                const float tn = a.T * s.seg[w][lane].x;   // (a 4-byte read outside warp 0)
                if (tn < c.stop_t) {
                    rw = w;
                    tin = a.T;
                    break;
                }
                if (wid == 0) {
                    const float4 g = s.seg[w][lane];
                    a.cr += a.T * g.y;
                    a.cg += a.T * g.z;
                    a.cb += a.T * g.w;
                }
                a.T = tn;
            }
        }
        // 5. pixels retiring inside this warp's segment: exact re-composite from their true T
        uint32_t mine = __ballot_sync(0xffffffffu, rw == wid);
        while (mine) {
            const int pl = __ffs(mine) - 1;
            mine &= mine - 1u;
            const uint32_t cov = __ballot_sync(0xffffffffu, (fp >> pl) & 1u);
            const float T_in = __shfl_sync(0xffffffffu, tin, pl);
            const float qx = __shfl_sync(0xffffffffu, c.fpx, pl), qy = __shfl_sync(0xffffffffu, c.fpy, pl);
            float sr, sg, sb, sc, T_out;
            pixel_entry_parallel(c, s.recs[wid][slot], cov, T_in, qx, qy, m.x, sr, sg, sb, sc, T_out);
            if (lane == pl) s.fin[pl] = make_float4(T_out, sr, sg, sb);   // warp 0 adds its colour
        }
        if (rw >= 0) {
            a.done = true;
            retired_here = true;
        }
        __syncwarp();   // the slot is refilled by a later chunk
        blended++;
    }
    cp_async_wait<0>();
    __syncwarp();
#ifdef SC_BLEND_STATS
    d.meta = min(mbase, end) - start;
#endif
}

// Frame path, persistent: every warp repeatedly takes the next (16x16 tile, 8x4
// block) list from an atomic ticket over the LPT order (longest lists first) and
// walks it.  No CTA barrier and no CTA-wide lifetime: a warp whose list is short
// takes the next one at once, so the SM's warp slots stay busy until the queue
// drains (one CTA per tile kept a CTA resident until its longest list ended:
// ~17 % warps active).  Per list the walk is the same as k_blend's, so images
// are bit-identical.
template <int REC>
#ifndef SC_BLEND_CPS
#define SC_BLEND_CPS 6   // 72 registers, no spills (7 CTAs fit); 8 per SM at 64 spilled: -0.2 %
#endif
__global__ void __launch_bounds__(kBlendWarps * 32, SC_BLEND_CPS) k_blend_blocks(
    const sc_splat *__restrict__ splats, int64_t n_splats, const uint32_t *__restrict__ boff,
    const uint32_t *__restrict__ vals, const uint32_t *__restrict__ keys, const uint32_t *__restrict__ task_order,
    int64_t n_tasks, unsigned long long *ticket, int width, int height, int n_tx, float stop_t, float bg_r,
    float bg_g, float bg_b, float *image, float *trans, float *csum, float *cmax)
{
    extern __shared__ float4 s_dyn[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WalkCtx c;
    c.splats = splats;
    c.n_splats = n_splats;
    c.vals = vals;
    c.keys = keys;
    c.wins = nullptr;
    c.blocks = 1;
    c.stop_t = stop_t;
    c.record = REC;   // compile-time: the non-recording kernels carry no contribution code
    c.cmax = cmax;
    c.lane = lane;
    char *wbase = reinterpret_cast<char *>(s_dyn) + wid * kWarpSmem;
    c.hq = reinterpret_cast<uint2 *>(wbase);
    c.stage = reinterpret_cast<uint2 *>(wbase + kHQBytesW);
    c.recs = reinterpret_cast<float4 *>(wbase + kHQBytesW + kStageMetaBytesW);
#ifdef SC_BLEND_STATS
    WalkStats d{0, 0, 0, 0, 0};
#endif
    // phase 1: the long lists at the head of the LPT order, one CTA each
    const int64_t n_coop = (int64_t)*reinterpret_cast<volatile unsigned long long *>(ticket + 2);
    if (n_coop > 0) {
        CoopSmem &s = *reinterpret_cast<CoopSmem *>(s_dyn);
        // code_mask(c) = cols(x0, x1) * rows(y0, y1): cols = code_mask(c & 63) (row 0 only), rows = code_mask of
        // the row bits with x0 = x1 = 0 (column 0 only)
        if (threadIdx.x < 64) s.mask_x[threadIdx.x] = code_mask(threadIdx.x);
        if (threadIdx.x < 16) s.mask_y[threadIdx.x] = code_mask(threadIdx.x << 6);
        for (int it = 0;; it++) {
            if (threadIdx.x == 0) s.ticket[it & 1] = (uint32_t)atomicAdd(ticket + 1, 1ull);
            __syncthreads();
            const int64_t t = s.ticket[it & 1];
            if (t >= n_coop) break;
            const uint32_t blk = __ldg(task_order + t);
            const int tile = (int)(blk >> 3), b = (int)(blk & 7u);
            const int tyi = tile / n_tx, txi = tile - tyi * n_tx;
            c.gx0 = txi * kTile + (b & 1) * 8;
            c.gy0 = tyi * kTile + (b >> 1) * 4;
            c.bx1 = c.gx0 + 7;
            c.by1 = c.gy0 + 3;
            const int px = c.gx0 + (lane & 7), py = c.gy0 + (lane >> 3);
            const bool inside = px < width && py < height;
            c.fpx = (float)px;
            c.fpy = (float)py;
            PixAcc a{1.0f, 0.0f, 0.0f, 0.0f, 0.0f, !inside};
            bool retired_here = false;
            coop_list(c, s, wid, __ldg(boff + blk), __ldg(boff + blk + 1), a, retired_here SC_WS_ARG);
#ifdef SC_BLEND_STATS
            if (threadIdx.x == 0 && blk < kDbgTiles * 8) {
                g_blend_used[2 * blk] = __ldg(boff + blk + 1) - __ldg(boff + blk);
                g_blend_used[2 * blk + 1] = (unsigned int)d.meta;
            }
#endif
            __syncthreads();   // s.fin complete
            if (wid == 0 && inside) {
                if (retired_here) {   // warp 0's colour stopped before the retiring segment
                    const float4 f = s.fin[lane];
                    a.T = f.x;
                    a.cr += f.y;
                    a.cg += f.z;
                    a.cb += f.w;
                }
                const int64_t p = (int64_t)py * width + px;
                image[3 * p + 0] = a.cr + a.T * bg_r;
                image[3 * p + 1] = a.cg + a.T * bg_g;
                image[3 * p + 2] = a.cb + a.T * bg_b;
                trans[p] = a.T;
            }
        }
        // every warp has read the last ticket before any warp's phase-2 queues (which reuse
        // these bytes) are written (racecheck: a WAR on s.ticket without this barrier)
        __syncthreads();
    }
    // phase 2: the remaining lists, one warp each
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = (unsigned long long)n_coop + atomicAdd(ticket, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int64_t)t >= n_tasks) break;
        const uint32_t blk = __ldg(task_order + t);   // block id = 8 tile + b
        const int tile = (int)(blk >> 3), b = (int)(blk & 7u);
        const int tyi = tile / n_tx, txi = tile - tyi * n_tx;
        c.gx0 = txi * kTile + (b & 1) * 8;
        c.gy0 = tyi * kTile + (b >> 1) * 4;
        c.bx1 = c.gx0 + 7;
        c.by1 = c.gy0 + 3;
        const int px = c.gx0 + (lane & 7), py = c.gy0 + (lane >> 3);
        const bool inside = px < width && py < height;
        c.fpx = (float)px;
        c.fpy = (float)py;
        PixAcc a{1.0f, 0.0f, 0.0f, 0.0f, 0.0f, !inside};
        walk_list(c, __ldg(boff + blk), __ldg(boff + blk + 1), a SC_WS_ARG);
#ifdef SC_BLEND_STATS
        if (lane == 0 && blk < kDbgTiles * 8) {
            g_blend_used[2 * blk] = __ldg(boff + blk + 1) - __ldg(boff + blk);
            g_blend_used[2 * blk + 1] = (unsigned int)d.meta;
        }
#endif
        if (inside) {
            const int64_t p = (int64_t)py * width + px;
            image[3 * p + 0] = a.cr + a.T * bg_r;
            image[3 * p + 1] = a.cg + a.T * bg_g;
            image[3 * p + 2] = a.cb + a.T * bg_b;
            trans[p] = a.T;
            if (REC && csum) csum[p] = a.cs;
        }
    }
}

// LPT dispatch order: heavier tiles first, bucketed by floor(log2(weight)),
// weight = the longest list among the tile's `stride` lists (the tile's
// critical path); the order inside a bucket is irrelevant to the result.
__device__ __forceinline__ uint32_t tile_weight(const uint32_t *off, int64_t t, int stride)
{
    uint32_t w = 0;
    for (int b = 0; b < stride; b++) w = max(w, off[stride * t + b + 1] - off[stride * t + b]);
    return w;
}

__global__ void __launch_bounds__(1024) k_tile_order(const uint32_t *off, int64_t tile_base, int64_t n_tiles,
                                                     int stride, uint32_t *order, unsigned long long *n_long,
                                                     int long_log2)
{
    __shared__ uint32_t hist[33], base[33];
    constexpr int kPer = 16;   // tiles per thread kept in registers (one weight pass)
    if (threadIdx.x < 33) hist[threadIdx.x] = 0;
    __syncthreads();
    uint32_t bucket[kPer];
    for (int64_t t0 = 0; t0 < n_tiles; t0 += (int64_t)blockDim.x * kPer) {
#pragma unroll
        for (int q = 0; q < kPer; q++) {
            const int64_t t = t0 + (int64_t)q * blockDim.x + threadIdx.x;
            uint32_t b = 0xFFFFFFFFu;
            if (t < n_tiles) {
                const uint32_t c = tile_weight(off, tile_base + t, stride);
                b = c ? 32 - __clz(c) : 0;
            }
            bucket[q] = b;
            // warp-aggregated histogram: one shared atomic per distinct bucket in the warp
            const uint32_t peers = __match_any_sync(0xffffffffu, b);
            if (b != 0xFFFFFFFFu && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[b], __popc(peers));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int b = 32; b >= 0; b--) {
            base[b] = run;
            run += hist[b];
        }
        // lists of >= 2^long_log2 entries (buckets > long_log2) lead the order
        if (n_long) *n_long = long_log2 >= 0 && long_log2 < 32 ? base[long_log2] : 0;
    }
    __syncthreads();
    for (int64_t t0 = 0; t0 < n_tiles; t0 += (int64_t)blockDim.x * kPer) {
        const bool single = n_tiles <= (int64_t)blockDim.x * kPer;   // weights still in registers
#pragma unroll
        for (int q = 0; q < kPer; q++) {
            const int64_t t = t0 + (int64_t)q * blockDim.x + threadIdx.x;
            uint32_t b = 0xFFFFFFFFu;
            if (t < n_tiles) {
                if (single) {
                    b = bucket[q];
                } else {
                    const uint32_t c = tile_weight(off, tile_base + t, stride);
                    b = c ? 32 - __clz(c) : 0;
                }
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, b);
            uint32_t slot = 0;
            const int leader = __ffs(peers) - 1;
            if (b != 0xFFFFFFFFu && (int)(threadIdx.x & 31) == leader) slot = atomicAdd(&base[b], __popc(peers));
            slot = __shfl_sync(0xffffffffu, slot, leader) + __popc(peers & lanemask_lt());
            if (b != 0xFFFFFFFFu) order[slot] = (uint32_t)(tile_base + t);
        }
    }
}

// Frame path: the same LPT order over the (tile, block) lists, built by many CTAs
// (the single-CTA k_tile_order was ~80 us on the frame's critical path): a bucket
// histogram, then every list takes a slot in its bucket from an atomic cursor (the
// order inside a bucket is arbitrary; each list's result does not depend on it).
__device__ __forceinline__ uint32_t list_bucket(const uint32_t *off, int64_t t)
{
    const uint32_t c = off[t + 1] - off[t];
    return c ? 32 - __clz(c) : 0;
}

__global__ void k_order_hist(const uint32_t *__restrict__ off, int64_t base, int64_t n, unsigned int *hist)
{
    __shared__ unsigned int h[33];
    if (threadIdx.x < 33) h[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[list_bucket(off, base + t)], 1u);
    __syncthreads();
    if (threadIdx.x < 33 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void k_order_scatter(const uint32_t *__restrict__ off, int64_t base, int64_t n, const unsigned int *hist,
                                unsigned int *cursor, uint32_t *order, unsigned long long *n_long, int long_log2)
{
    __shared__ unsigned int s_base[33];
    if (threadIdx.x == 0) {
        unsigned int run = 0;
        for (int b = 32; b >= 0; b--) {   // heavier buckets first
            s_base[b] = run;
            run += hist[b];
        }
        if (blockIdx.x == 0 && n_long) *n_long = long_log2 >= 0 && long_log2 < 32 ? s_base[long_log2] : 0;
    }
    __syncthreads();
    for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x; t0 < n; t0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = t0 + threadIdx.x;
        const uint32_t b = t < n ? list_bucket(off, base + t) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(peers) - 1;
        uint32_t slot = 0;
        if (b != 0xFFFFFFFFu && (int)(threadIdx.x & 31) == leader) slot = atomicAdd(&cursor[b], __popc(peers));
        slot = __shfl_sync(0xffffffffu, slot, leader) + __popc(peers & lanemask_lt());
        if (b != 0xFFFFFFFFu) order[s_base[b] + slot] = (uint32_t)(base + t);
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

// Threshold (log2 entries) of the lists walked by a whole CTA; the environment
// variable SPLATCULL_B200_LONG_LIST_LOG2 overrides it (tests force the CTA walk on
// small scenes with it; a value >= 32 disables it).
static int long_list_log2()
{
    const char *e = getenv("SPLATCULL_B200_LONG_LIST_LOG2");
    return e && *e ? atoi(e) : SC_COOP_LOG2;
}

template <int REC>
static cudaError_t blend_impl(const sc_splat *splats, const BlendLists &lists, const sc_camera &cam, const sc_opts &opts,
                              const sc_frame_out &out, int64_t n_splats, uint32_t *task_order, cudaStream_t st)
{
    constexpr int kSmem = (int)(kBlendWarps * kWarpSmem);
    {
        cudaError_t e = smem_attr_once(reinterpret_cast<const void *>(k_blend<REC>), kSmem);
        if (e != cudaSuccess) return e;
    }
    // frame path: 16x16 CTA tiles of 8 blocks; tile lists: the reference's tile size
    const int ts = lists.blocks ? kTile : opts.tile_size;
    const int n_tx = (cam.width + ts - 1) / ts;
    const int nbx = (ts + 7) / 8, nblk = nbx * ((ts + 3) / 4);
    const int ngroups = (nblk + kBlendWarps - 1) / kBlendWarps;
    const Band band = band_of(opts, cam.height, ts);   // only the band's tiles are blended (and written)
    const int64_t tile_base = (int64_t)band.t0 * n_tx, n_tiles = (int64_t)(band.t1 - band.t0) * n_tx;
    if (n_tiles <= 0) return cudaSuccess;
#ifndef SC_BLEND_PERSIST
#define SC_BLEND_PERSIST 1
#endif
    if (SC_BLEND_PERSIST && lists.blocks && task_order && lists.ctr) {
        // frame path: persistent warps over the (tile, block) lists, longest first
        cudaError_t e = smem_attr_once(reinterpret_cast<const void *>(k_blend_blocks<REC>), kSmem);
        if (e != cudaSuccess) return e;
        static int cps_cache[64];
        int dev = 0;
        cudaGetDevice(&dev);
        int cps = (dev >= 0 && dev < 64) ? cps_cache[dev] : 0;
        if (cps <= 0) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cps, k_blend_blocks<REC>, kBlendWarps * 32, kSmem);
            if (e != cudaSuccess) return e;
            cps = std::max(cps, 1);
            if (dev >= 0 && dev < 64) cps_cache[dev] = cps;
        }
        const int64_t n_tasks = 8 * n_tiles;
        // ticket[0]: next short list (per warp), [1]: next long list (per CTA), [2]: number of long lists
        unsigned long long *ticket = &lists.ctr->blend_next;   // [0] short lists, [1] long lists, [2] n_long
        unsigned int *hist = lists.ctr->order_hist, *cursor = lists.ctr->order_cursor;
        const int ogrid = (int)std::max<int64_t>(1, std::min<int64_t>((n_tasks + 255) / 256, (int64_t)sm_count()));
        SC_LAUNCH(k_order_hist, ogrid, 256, 0, st, lists.offsets, 8 * tile_base, n_tasks, hist);
        SC_LAUNCH(k_order_scatter, ogrid, 256, 0, st, lists.offsets, 8 * tile_base, n_tasks, hist, cursor, task_order,
                  ticket + 2, REC ? -1 : long_list_log2());
        const int grid = (int)std::min<int64_t>((n_tasks + kBlendWarps - 1) / kBlendWarps, (int64_t)sm_count() * cps);
        SC_LAUNCH(k_blend_blocks<REC>, grid, kBlendWarps * 32, kSmem, st, splats, n_splats, lists.offsets, lists.vals,
                  lists.keys, task_order, n_tasks, ticket, cam.width, cam.height, n_tx,
                  (float)opts.stop_transmittance, (float)opts.background[0], (float)opts.background[1],
                  (float)opts.background[2], out.image, out.trans,
                  out.contrib_sum, out.contrib_max);
        return cudaGetLastError();
    }
    if (n_tiles * ngroups > 0x7FFFFFFFll) return cudaErrorInvalidValue;
    if (task_order)
        SC_LAUNCH(k_tile_order, 1, 1024, 0, st, lists.offsets, tile_base, n_tiles, lists.blocks ? 8 : 1, task_order,
                  (unsigned long long *)nullptr, -1);
    SC_LAUNCH(k_blend<REC>, (int)(n_tiles * ngroups), kBlendWarps * 32, kSmem, st, splats, n_splats, lists.offsets, lists.vals,
              lists.keys, lists.wins, lists.blocks ? 1 : 0, task_order, (int)tile_base, cam.width, cam.height, n_tx,
              ts, nbx, nblk, ngroups,
              (float)opts.stop_transmittance, (float)opts.background[0], (float)opts.background[1],
              (float)opts.background[2], out.image, out.trans, out.contrib_sum,
              out.contrib_max);
    return cudaGetLastError();
}

cudaError_t launch_blend(const sc_splat *splats, const BlendLists &lists, const sc_camera &cam, const sc_opts &opts,
                         const sc_frame_out &out, int64_t n_splats, uint32_t *task_order, cudaStream_t st)
{
    return opts.record_contributions ? blend_impl<1>(splats, lists, cam, opts, out, n_splats, task_order, st)
                                     : blend_impl<0>(splats, lists, cam, opts, out, n_splats, task_order, st);
}

// Visibility labels (sc/sampling.py:206-213): bit i of the little-endian word
// array |= (contribution_max[i] > 0); a warp packs 32 splats with one ballot.
__global__ void k_labels_or(const float *cmax, int64_t n, uint32_t *bits)
{
    const int lane = threadIdx.x & 31;
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + lane;
        const uint32_t w = __ballot_sync(0xffffffffu, i < n && cmax[i] > 0.0f);
        if (lane == 0 && w) bits[base >> 5] |= w;
    }
}

cudaError_t launch_labels_or(const float *cmax, int64_t n, uint32_t *bits, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 8));
    SC_LAUNCH(k_labels_or, grid, 256, 0, st, cmax, n, bits);
    return cudaGetLastError();
}

cudaError_t launch_count_used(const float *cmax, const unsigned long long *n_dev, int64_t n_max,
                              sc_frame_stats *stats, cudaStream_t st)
{
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_max + 255) / 256, (int64_t)sm_count() * 8));
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
// [n_blocks][2] = (list length, entries streamed before the walk stopped) of the last frame
extern "C" __attribute__((visibility("default"))) int sc_debug_blend_used(unsigned int *host, int64_t n_blocks)
{
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, sc::g_blend_used) != cudaSuccess) return 2;
    const size_t bytes = sizeof(unsigned int) * 2 * (size_t)std::min<int64_t>(n_blocks, 8 * sc::kDbgTiles);
    return cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 2;
}
#endif
