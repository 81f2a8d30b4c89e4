// Stages (a) + (b): per-instance bounding-sphere cull, per-(instance, gaussian)
// frustum test, d_near gate and the fused tcgen05 visibility MLP, with an
// order-preserving compaction of survivors (per-chunk staging, scan, k_compact).
//
// Compiled with -fmad=false: the frustum / gate arithmetic is float64 and must
// reproduce the oracle (oracle/sc_oracle.c:orc_scene_cull) bit for bit.
//
// Reference semantics: SPEC.md:344-361 (local_inputs, render_composed steps
// 1-2), SPEC.md:378-379 (margin, below-d_near rule), PAPER.md:186-204 (Eq. 2).
#include <algorithm>

#include "tc05.cuh"

namespace sc {

// ---------------------------------------------------------------------------
// Per-instance prep: Eq. 2 factor, local camera forward, conservative
// bounding-sphere test and the chunk prefix.  One CTA of 1024 threads.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_prep(sc_scene scene, sc_camera cam, sc_opts opts, Ws ws,
                                               sc_frame_stats *stats)
{
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_running;
    __shared__ unsigned long long s_pairs, s_vis, s_dlo, s_dhi;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // passed splats have depth > near; non-negative doubles order as their bits
    const double d_floor = fmax(cam.near_, 0.0);
    if (tid == 0) {
        s_running = 0;
        s_pairs = 0;
        s_vis = 0;
        s_dlo = (unsigned long long)__double_as_longlong(INFINITY);
        s_dhi = 0ull;
    }
    __syncthreads();
    const double f = cam.focal;
    const double cxp = (double)(cam.width - 1) / 2.0, cyp = (double)(cam.height - 1) / 2.0;
    const int ts = opts.tile_size;
    const double TW = (double)(ts * ((cam.width + ts - 1) / ts));
    const Band band = band_of(opts, cam.height, ts);
    const bool banded = opts.band_y1 > 0;
    const double PAD = margin_pad(opts.dilation);
    for (int64_t base = 0; base < scene.n_instances; base += 1024) {
        const int64_t i = base + tid;
        uint32_t nch = 0;
        unsigned long long t_dlo = (unsigned long long)__double_as_longlong(INFINITY), t_dhi = 0ull, t_pairs = 0ull,
                           t_vis = 0ull;
        if (i < scene.n_instances) {
            const sc_instance_rec &in = scene.instances[i];
            const sc_asset_rec &a = scene.assets[in.asset];
            InstFrame fr;
            fr.corr = (a.model >= 0) ? (a.f_train / cam.focal) / in.s : 0.0;
            for (int k = 0; k < 3; k++)
                fr.fwd_local[k] = (float)(in.R[k] * cam.rot[6] + in.R[3 + k] * cam.rot[7] + in.R[6 + k] * cam.rot[8]);
            {
                const double d0 = in.t[0] - cam.pos[0], d1 = in.t[1] - cam.pos[1], d2 = in.t[2] - cam.pos[2];
                for (int k = 0; k < 3; k++) fr.cam_local[k] = (float)(in.R[k] * d0 + in.R[3 + k] * d1 + in.R[6 + k] * d2);
                fr.s = (float)in.s;
                const double span = a.d_far - a.d_near;
                fr.dn_a = (float)(2.0 * fr.corr / span);
                fr.dn_b = (float)(-2.0 * a.d_near / span - 1.0);
            }
            int vis = a.count > 0;
            // sphere around the instance covering every instanced mean, with slack
            // for the f32 rounding of instanced means
            const double tmax = fmax(fabs(in.t[0]), fmax(fabs(in.t[1]), fabs(in.t[2])));
            const double rho = in.s * a.bound_local * (1.0 + 1e-6) + 1e-6 * (2.0 * tmax + in.s * a.bound_local) + 1e-9;
            double cx, cy, cz;
            cam_xyz(cam, in.t[0], in.t[1], in.t[2], cx, cy, cz);
            if (opts.frustum_mode != SC_FRUSTUM_OFF && vis) {
                if (cz + rho <= cam.near_) vis = 0;
                double mg = 0.0, pad = 0.0, xlo = 0.0, xhi = (double)(cam.width - 1), ylo = 0.0,
                       yhi = (double)(cam.height - 1);
                if (opts.frustum_mode == SC_FRUSTUM_MARGIN) {
                    mg = 3.0 * f * opts.frustum_G * in.s * a.sigma_max * (1.0 + 1e-6);
                    pad = PAD;
                    xhi = TW;
                    ylo = (double)band.y0;
                    yhi = (double)band.y1;
                }
                // low side:  f t + (c + pad - lo) z + mg >= 0 must be reachable
                double kl = cxp + pad - xlo;
                if (f * cx + kl * cz + mg + rho * sqrt(f * f + kl * kl) < 0.0) vis = 0;
                double kh = cxp - pad - xhi;
                if (f * cx + kh * cz - mg - rho * sqrt(f * f + kh * kh) > 0.0) vis = 0;
                kl = cyp + pad - ylo;
                if (f * cy + kl * cz + mg + rho * sqrt(f * f + kl * kl) < 0.0) vis = 0;
                kh = cyp - pad - yhi;
                if (f * cy + kh * cz - mg - rho * sqrt(f * f + kh * kh) > 0.0) vis = 0;
            }
            if (banded && opts.frustum_mode != SC_FRUSTUM_MARGIN && vis) {   // band rows, margin style
                const double mgb = 3.0 * f * opts.frustum_G * in.s * a.sigma_max * (1.0 + 1e-6);
                if (cz + rho <= cam.near_) vis = 0;
                double kl = cyp + PAD - (double)band.y0;
                if (f * cy + kl * cz + mgb + rho * sqrt(f * f + kl * kl) < 0.0) vis = 0;
                double kh = cyp - PAD - (double)band.y1;
                if (f * cy + kh * cz - mgb - rho * sqrt(f * f + kh * kh) > 0.0) vis = 0;
            }
            // Uniform instances (every pair decided the same way) skip the per-pair f64
            // tests in k_cull.  inside: the sphere lies strictly inside z > near and the
            // image-plane region the per-pair test accepts unconditionally
            // ([0, TW) x [0, TH) in margin mode, where rb >= 3 px more is tolerated;
            // [1e-3, W-1-1e-3]^2 in strict mode) -- the per-pair f64 rounding (~1e-12 px)
            // cannot flip such a pair.
            int inside = 0, gate = -1;
            if (vis) {
                const double rr = rho * (1.0 + 1e-6) + 1e-9;
                // plane  f x + (c - b) z >= 0  (mx >= b)  and  -(f x + (c - b) z) >= 0  (mx <= b)
                auto dist_ge = [&](double px, double pz, double k, double sign) {
                    const double v = sign * (f * px + k * pz);
                    return v > rr * sqrt(f * f + k * k) * (1.0 + 1e-9);
                };
                const bool front = cz - rr > cam.near_ * (1.0 + 1e-9) + 1e-12;
                if (opts.frustum_mode == SC_FRUSTUM_OFF) {
                    inside = 1;
                } else {
                    const bool strict = opts.frustum_mode == SC_FRUSTUM_STRICT;
                    const double lo = strict ? 1e-3 : 0.0;
                    const double hx = strict ? (double)(cam.width - 1) - 1e-3 : TW;
                    const double ly = strict ? 1e-3 : (double)band.y0;
                    const double hy = strict ? (double)(cam.height - 1) - 1e-3 : (double)band.y1;
                    inside = front && dist_ge(cx, cz, cxp - lo, 1.0) && dist_ge(cx, cz, cxp - hx, -1.0) &&
                             dist_ge(cy, cz, cyp - ly, 1.0) && dist_ge(cy, cz, cyp - hy, -1.0);
                }
                // the band rows (margin style, rb >= 3 px of slack) in the other modes
                if (banded && opts.frustum_mode != SC_FRUSTUM_MARGIN)
                    inside = inside && front && dist_ge(cy, cz, cyp - (double)band.y0, 1.0) &&
                             dist_ge(cy, cz, cyp - (double)band.y1, -1.0);
                if (a.model >= 0 && opts.use_mlp) {
                    const double dc = sqrt((in.t[0] - cam.pos[0]) * (in.t[0] - cam.pos[0]) +
                                           (in.t[1] - cam.pos[1]) * (in.t[1] - cam.pos[1]) +
                                           (in.t[2] - cam.pos[2]) * (in.t[2] - cam.pos[2]));
                    const double rr = rho * (1.0 + 1e-6) + 1e-9;
                    if ((dc - rr) * fr.corr > a.d_near * (1.0 + 1e-9)) gate = 1;
                    else if ((dc + rr) * fr.corr < a.d_near * (1.0 - 1e-9)) gate = 0;
                } else {
                    gate = 0;
                }
            }
            fr.inside = inside;
            fr.gate = gate;
            if (vis) {   // depth range of every instanced mean of a visible instance (frame-path sort keys)
                const double lo = fmax(cz - rho * (1.0 + 1e-9), d_floor);
                const double hi = fmax(cz + rho * (1.0 + 1e-9), lo);
                t_dlo = (unsigned long long)__double_as_longlong(lo);
                t_dhi = (unsigned long long)__double_as_longlong(hi);
            }
            fr.visible = vis;
            nch = vis ? (uint32_t)((a.count + kChunk - 1) / kChunk) : 0u;
            fr.n_chunks = nch;
            fr.chunk_begin = 0;
            ws.inst[i] = fr;
            if (vis) {
                t_pairs = (unsigned long long)a.count;
                t_vis = 1ull;
            }
        }
        // warp reductions, one shared atomic per warp (1,000 threads on one address serialise)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            t_dlo = min(t_dlo, __shfl_xor_sync(0xffffffffu, t_dlo, o));
            t_dhi = max(t_dhi, __shfl_xor_sync(0xffffffffu, t_dhi, o));
            t_pairs += __shfl_xor_sync(0xffffffffu, t_pairs, o);
            t_vis += __shfl_xor_sync(0xffffffffu, t_vis, o);
        }
        if (lane == 0) {
            if (t_vis) {
                atomicMin(&s_dlo, t_dlo);
                atomicMax(&s_dhi, t_dhi);
                atomicAdd(&s_pairs, t_pairs);
                atomicAdd(&s_vis, t_vis);
            }
        }
        // block exclusive scan of nch
        uint32_t x = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_warp[lane] = w;
        }
        __syncthreads();
        const uint32_t excl = s_running + (wid ? s_warp[wid - 1] : 0u) + x - nch;
        if (i < scene.n_instances) ws.inst[i].chunk_begin = excl;
        __syncthreads();
        if (tid == 0) s_running += s_warp[31];
        __syncthreads();
    }
    if (tid == 0) {
        // a scene with more pairs than the workspace was sized for (sc_scene.n_pairs
        // understated): cull nothing rather than write past the chunk arrays
        const bool fits = (int64_t)s_running <= ws.max_chunks;
        if (!fits) atomicOr((unsigned long long *)&stats->overflow, 8ull);
        ws.ctr->total_chunks = fits ? s_running : 0u;
        ws.ctr->chunk_ticket = 0;
        stats->instances_visible = (int64_t)s_vis;
        // frame-path depth keys: floor((tz - dmin) * scale) over [dmin, dmax] (k_project)
        const double dlo = __longlong_as_double((long long)s_dlo), dhi = __longlong_as_double((long long)s_dhi);
        ws.ctr->key_dmin = s_vis ? dlo : 0.0;
        ws.ctr->key_scale = (s_vis && dhi > dlo) ? 4294967040.0 / (dhi - dlo) : 0.0;
        stats->pairs_tested = (int64_t)s_pairs;
    }
}


// chunk -> owning instance: the last instance with chunk_begin <= chunk (one thread
// per chunk, binary search; invisible instances own no chunk and share their
// successor's chunk_begin, so "last" is the owner)
__global__ void k_chunk_map(const InstFrame *__restrict__ inst, int64_t n_inst, const Counters *ctr,
                            uint32_t *chunk_inst)
{
    const int64_t total = (int64_t)ctr->total_chunks;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < total; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n_inst;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (inst[mid].chunk_begin <= (uint32_t)c) lo = mid; else hi = mid;
        }
        chunk_inst[c] = (uint32_t)lo;
    }
}

// ---------------------------------------------------------------------------
// Cull + MLP.  Persistent CTAs of 128 threads take chunks of kChunk pairs of
// one instance from an atomic ticket.  Each 128-pair tile: thread = pair; f64
// frustum test on the f32-rounded instanced mean (B2/B3), Eq. 2 gate in f64, 16
// fp16 inputs into the smem A tile, tcgen05 MLP, survivor ballot into an smem
// list kept in pair order.  The chunk's list goes to its own staging slot;
// k_compact places it after its predecessors' (scan of the chunk counts), so
// no CTA waits on another (a decoupled look-back here stalled ~20 % of the time).
// ---------------------------------------------------------------------------
#ifndef SC_CULL_CPS
#define SC_CULL_CPS 12
#endif
__global__ void __launch_bounds__(kCullThreads, SC_CULL_CPS) k_cull(sc_scene scene, sc_camera cam, sc_opts opts, Ws ws,
                                                       sc_survivor *out, long long cap, sc_frame_stats *stats)
{
    __shared__ MlpSmem sm;
    __shared__ sc_instance_rec s_in;
    __shared__ sc_asset_rec s_as;
    __shared__ InstFrame s_fr;
    // the chunk's MLP-input constants, one broadcast 16-byte load each per pair: (s, cam_local),
    // (dn_a, dn_b, 1 / mean_scale, fwd_local[0]), fp16x2 (fwd_local[1], fwd_local[2])
    __shared__ float4 s_fc[2];
    __shared__ uint32_t s_fwd12;
    __shared__ uint16_t s_surv[kChunk];   // survivors of the chunk: offset from the chunk start
    constexpr int kCullWarps = kCullThreads / 32;
    constexpr int kSegs = kCullTilesPerChunk * kCullWarps, kSegPerLane = kSegs / 32;
    static_assert(kSegs % 32 == 0 && kChunk <= 65536, "one warp scans the chunk's segment counts; u16 offsets");
    __shared__ uint32_t s_wcnt[kCullTilesPerChunk * kCullWarps];   // survivors per (tile, warp) segment
    __shared__ uint32_t s_segoff[kCullTilesPerChunk * kCullWarps];
    __shared__ uint32_t s_chunk, s_inst, s_nc;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    mlp_setup(sm, tid);
    uint32_t phase = 0;
    int loaded_model = -1;
    uint32_t n_pass = 0, n_query = 0, n_cull = 0;   // per thread (< 2^32 pairs each)
    const unsigned long long total = ws.ctr->total_chunks;
    const double cxp = (double)(cam.width - 1) / 2.0, cyp = (double)(cam.height - 1) / 2.0;
    const int ts = opts.tile_size;
    const double TW = (double)(ts * ((cam.width + ts - 1) / ts));
    const Band band = band_of(opts, cam.height, ts);
    const bool banded = opts.band_y1 > 0;
    const double PAD = margin_pad(opts.dilation);
    const double BY0 = (double)band.y0, BY1 = (double)band.y1;   // whole image: [0, TH)

    // chunks are handed out by an atomic ticket (dynamic balance across CTAs)
    for (;;) {
        if (tid == 0) s_chunk = (uint32_t)atomicAdd(&ws.ctr->chunk_ticket, 1ull);
        __syncthreads();
        const uint32_t chunk = s_chunk;
        if (chunk >= total) break;
        for (int q = tid; q < kSegs; q += kCullThreads) s_wcnt[q] = 0;   // tiles past the chunk end stay empty
        if (wid == 0) {
            // the chunk's instance (k_chunk_map), then the warp copies the instance, its asset
            // and its frame records word by word (two load latencies)
            const int64_t lo = (int64_t)ws.chunk_inst[chunk];
            static_assert(sizeof(sc_instance_rec) % 4 == 0 && sizeof(sc_asset_rec) % 4 == 0 &&
                              sizeof(InstFrame) % 4 == 0, "word copies");
            const uint32_t *gi = reinterpret_cast<const uint32_t *>(scene.instances + lo);
            const uint32_t *gf = reinterpret_cast<const uint32_t *>(ws.inst + lo);
            uint32_t *si = reinterpret_cast<uint32_t *>(&s_in), *sf = reinterpret_cast<uint32_t *>(&s_fr);
            for (int w = lane; w < (int)(sizeof(sc_instance_rec) / 4); w += 32) si[w] = gi[w];
            for (int w = lane; w < (int)(sizeof(InstFrame) / 4); w += 32) sf[w] = gf[w];
            const int asset = scene.instances[lo].asset;
            const uint32_t *ga = reinterpret_cast<const uint32_t *>(scene.assets + asset);
            uint32_t *sa = reinterpret_cast<uint32_t *>(&s_as);
            for (int w = lane; w < (int)(sizeof(sc_asset_rec) / 4); w += 32) sa[w] = ga[w];
            __syncwarp();
            if (lane == 0) {
                s_inst = (uint32_t)lo;
                s_fc[0] = make_float4(s_fr.s, s_fr.cam_local[0], s_fr.cam_local[1], s_fr.cam_local[2]);
                s_fc[1] = make_float4(s_fr.dn_a, s_fr.dn_b, (float)s_as.inv_mean_scale, s_fr.fwd_local[0]);
                s_fwd12 = pack_h2(s_fr.fwd_local[1], s_fr.fwd_local[2]);
            }
        }
        __syncthreads();
        const int model = (opts.use_mlp && s_as.model >= 0) ? s_as.model : -1;
        if (model >= 0 && model != loaded_model) {
            mlp_load_weights(sm, scene.vis_weights + model, tid, kCullThreads);
            loaded_model = model;
            __syncthreads();
        }
        const int64_t j0 = (int64_t)(chunk - s_fr.chunk_begin) * kChunk;
        // pairs of the chunk: gaussians gbase + [0, nloc) of the asset (32-bit offsets in the loop)
        const int nloc = (int)(min(j0 + (int64_t)kChunk, s_as.count) - j0);
        const int64_t gbase = s_as.offset + j0;
        const float4 *mo_c = reinterpret_cast<const float4 *>(scene.mean_opa) + gbase;
        const uint4 *ft_c = reinterpret_cast<const uint4 *>(scene.features) + gbase;

        for (int t = 0; t < kCullTilesPerChunk; t++) {
            const int jt = t * kCullThreads;
            if (jt >= nloc) break;
            const int jl = jt + tid;   // pair offset in the chunk
            const bool active = jl < nloc;
            bool pass = false, queried = false;
            uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
            if (active) {
                const float4 mo = __ldg(mo_c + jl);
                // the f32 instanced mean (B2), only needed by the exact per-pair tests
                const bool need_mean = !s_fr.inside || (model >= 0 && s_fr.gate < 0);
                const float3 mw = need_mean ? inst_mean(s_in, mo.x, mo.y, mo.z) : make_float3(0.f, 0.f, 0.f);
                if (s_fr.inside) {
                    pass = true;   // k_prep: the whole instance sphere passes
                } else {
                    // exact per-pair test on the f32 instanced mean (B3), f64 as the oracle
                    const float smax = __ldg(scene.scale_smax + 4 * (gbase + jl) + 3);
                    double tx, ty, tz;
                    cam_xyz(cam, mw.x, mw.y, mw.z, tx, ty, tz);
                    if (opts.frustum_mode == SC_FRUSTUM_OFF) {
                        pass = true;   // only the band filter below
                    } else if (tz > cam.near_) {
                        const double mx = cam.focal * (tx / tz) + cxp;
                        const double my = cam.focal * (ty / tz) + cyp;
                        if (opts.frustum_mode == SC_FRUSTUM_STRICT) {
                            pass = mx >= 0.0 && mx <= (double)(cam.width - 1) && my >= 0.0 &&
                                   my <= (double)(cam.height - 1);
                        } else {
                            const double sigma_w = s_in.s * (double)smax;
                            const double rb = 3.0 * (cam.focal / tz) * sigma_w * opts.frustum_G + PAD;
                            pass = (mx + rb >= 0.0) && (mx - rb < TW) && (my + rb >= BY0) && (my - rb < BY1);
                        }
                    }
                    if (pass && banded && opts.frustum_mode != SC_FRUSTUM_MARGIN) {
                        // screen band: the same conservative margin test on the band rows
                        pass = false;
                        if (tz > cam.near_) {
                            const double my = cam.focal * (ty / tz) + cyp;
                            const double rb = 3.0 * (cam.focal / tz) * (s_in.s * (double)smax) * opts.frustum_G + PAD;
                            pass = (my + rb >= BY0) && (my - rb < BY1);
                        }
                    }
                }
                if (pass && model >= 0) {
                    if (s_fr.gate >= 0) {
                        queried = s_fr.gate == 1;   // k_prep: uniform over the instance sphere
                    } else {                        // exact Eq. 2 gate on the f32 instanced mean
                        const double dx = (double)mw.x - cam.pos[0], dy = (double)mw.y - cam.pos[1],
                                     dz = (double)mw.z - cam.pos[2];
                        queried = sqrt(dx * dx + dy * dy + dz * dz) * s_fr.corr >= s_as.d_near;
                    }
                    if (queried) {
                        // MLP inputs in the instance frame, f32 (they are rounded to fp16):
                        // R^T (m' - c) = s m + R^T (t - c)
                        const float4 fa = s_fc[0], fb = s_fc[1];
                        const float px = fmaf(fa.x, mo.x, fa.y);
                        const float py = fmaf(fa.x, mo.y, fa.z);
                        const float pz = fmaf(fa.x, mo.z, fa.w);
                        const float d2 = fmaf(px, px, fmaf(py, py, pz * pz));
                        const float rinv = rsqrtf(d2);
                        const float d_r = d2 * rinv;
                        const float dn = fminf(fmaxf(fmaf(d_r, fb.x, fb.y), -1.0f), 1.0f);
                        const float ims = fb.z;
                        lo = make_uint4(pack_h2(mo.x * ims, mo.y * ims), pack_h2(mo.z * ims, px * rinv),
                                        pack_h2(py * rinv, pz * rinv), pack_h2(dn, fb.w));
                        const uint4 feat = __ldg(ft_c + jl);
                        hi = make_uint4(s_fwd12, feat.x, feat.y, feat.z);
                    }
                }
            }
            bool keep = pass;
            if (model >= 0) {
                mlp_store_row(sm, tid, lo, hi);
                float logit;
                if (mlp_tile(sm, tid, phase, queried, &logit) && queried && !(logit >= s_as.logit_threshold))
                    keep = false;
            }
            n_pass += pass;
            n_query += queried;
            n_cull += (pass && !keep);
            // warp-local ordered compaction: segment (t, w) of the chunk, no CTA barrier
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) s_surv[t * kCullThreads + wid * 32 + __popc(bal & lanemask_lt())] = (uint16_t)jl;
            if (lane == 0) s_wcnt[t * kCullWarps + wid] = __popc(bal);
        }
        // chunk order = (tile, warp)-major: scan the 32 segment counts (one warp)
        __syncthreads();
        if (wid == 0) {   // lane: segments [kSegPerLane lane, kSegPerLane (lane + 1))
            uint32_t c[kSegPerLane], sum = 0;
#pragma unroll
            for (int q = 0; q < kSegPerLane; q++) {
                c[q] = s_wcnt[kSegPerLane * lane + q];
                sum += c[q];
            }
            uint32_t x = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            uint32_t run = x - sum;
#pragma unroll
            for (int q = 0; q < kSegPerLane; q++) {
                s_segoff[kSegPerLane * lane + q] = run;
                run += c[q];
            }
            if (lane == 31) s_nc = x;
        }
        __syncthreads();
        const uint32_t n_c = s_nc;

        // the chunk's survivors go to its staging slot (no wait on other chunks: their
        // order-preserving placement is a scan over the chunk counts + k_compact)
        if (tid == 0) {
            ws.chunk_cnt[chunk] = n_c;
            ws.chunk_state[chunk] = ((unsigned long long)s_inst << 32) | (uint32_t)(chunk - s_fr.chunk_begin);
        }
        uint16_t *stage = ws.chunk_stage + (size_t)chunk * kChunk;
        for (int t = 0; t < kCullTilesPerChunk; t++) {   // warp w copies its segments
            const int seg = t * kCullWarps + wid;
            if ((uint32_t)lane < s_wcnt[seg]) stage[s_segoff[seg] + lane] = s_surv[t * kCullThreads + wid * 32 + lane];
        }
    }
    // stats
    n_pass = __reduce_add_sync(0xffffffffu, n_pass);
    n_query = __reduce_add_sync(0xffffffffu, n_query);
    n_cull = __reduce_add_sync(0xffffffffu, n_cull);
    if (lane == 0) {
        if (n_pass) atomicAdd((unsigned long long *)&stats->frustum_passed, (unsigned long long)n_pass);
        if (n_query) atomicAdd((unsigned long long *)&stats->mlp_queried, (unsigned long long)n_query);
        if (n_cull) atomicAdd((unsigned long long *)&stats->mlp_culled, (unsigned long long)n_cull);
    }
    mlp_teardown(sm, tid);
}

// ---------------------------------------------------------------------------
// Survivor placement: chunk c's staged survivors land at the exclusive scan of
// the chunk counts (chunk order = pair order, so the list is the flat
// (asset, instance, gaussian) order of B1).  One warp per chunk.
// ---------------------------------------------------------------------------
__global__ void k_compact(const unsigned long long *__restrict__ chunk_state, const uint32_t *__restrict__ chunk_off,
                          const uint16_t *__restrict__ stage, const unsigned long long *n_chunks_dev,
                          const unsigned long long *total_dev, sc_survivor *out, long long cap,
                          sc_frame_stats *stats)
{
    const int64_t n_chunks = (int64_t)*n_chunks_dev;
    const int64_t total = (int64_t)*total_dev;
    if (blockIdx.x == 0 && threadIdx.x == 0 && total > cap) atomicOr((unsigned long long *)&stats->overflow, 1ull);
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < n_chunks; c += n_warps) {
        const int64_t o0 = chunk_off[c];
        const int64_t n = (c + 1 < n_chunks ? (int64_t)chunk_off[c + 1] : total) - o0;
        const unsigned long long cs = chunk_state[c];
        const uint32_t inst = (uint32_t)(cs >> 32);
        const uint32_t j0 = (uint32_t)cs * (uint32_t)kChunk;
        const uint16_t *src = stage + (size_t)c * kChunk;
        for (int64_t i = lane; i < n; i += 32) {
            if (o0 + i < cap) {
                sc_survivor sv;
                sv.inst = inst;
                sv.gid = j0 + src[i];
                out[o0 + i] = sv;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Batched forward on materialised fp32 inputs (config-4 sweep, nn.forward).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 12) k_vis_forward(const sc_vis_weights *w, const float *x, int64_t n,
                                                         float *logits)
{
    __shared__ MlpSmem sm;
    const int tid = threadIdx.x;
    mlp_setup(sm, tid);
    mlp_load_weights(sm, w, tid, 128);
    __syncthreads();
    uint32_t phase = 0;
    const int64_t n_tiles = (n + 127) / 128;
    // the next tile's row is loaded (and packed to fp16) while the current tile runs the MLP
    auto load = [&](int64_t tile, uint4 &lo, uint4 &hi) {
        const int64_t r = tile * 128 + tid;
        lo = make_uint4(0, 0, 0, 0);
        hi = lo;
        if (tile < n_tiles && r < n) {
            const float4 *row = reinterpret_cast<const float4 *>(x + r * 16);
            const float4 a = __ldcs(row), b = __ldcs(row + 1), c = __ldcs(row + 2), d = __ldcs(row + 3);
            lo = make_uint4(pack_h2(a.x, a.y), pack_h2(a.z, a.w), pack_h2(b.x, b.y), pack_h2(b.z, b.w));
            hi = make_uint4(pack_h2(c.x, c.y), pack_h2(c.z, c.w), pack_h2(d.x, d.y), pack_h2(d.z, d.w));
        }
    };
    uint4 lo, hi;
    load(blockIdx.x, lo, hi);
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t r = tile * 128 + tid;
        mlp_store_row(sm, tid, lo, hi);
        load(tile + gridDim.x, lo, hi);
        float lg = 0.0f;
        mlp_tile(sm, tid, phase, true, &lg);
        if (r < n) logits[r] = lg;
    }
    mlp_teardown(sm, tid);
}

// ---------------------------------------------------------------------------
// Feature MLP 14 -> 32 -> 32 -> 6 (once per asset, off the frame path).
// fp32 CUDA cores; output fp16 [n][8].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_encode_features(const float *params, const float *x, int64_t n,
                                                         uint16_t *feat)
{
    constexpr int P = 14 * 32 + 32 + 32 * 32 + 32 + 6 * 32 + 6;
    __shared__ float sp[P];
    for (int i = threadIdx.x; i < P; i += blockDim.x) sp[i] = params[i];
    __syncthreads();
    const float *W1 = sp, *b1 = W1 + 14 * 32, *W2 = b1 + 32, *b2 = W2 + 32 * 32, *W3 = b2 + 32, *b3 = W3 + 6 * 32;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        float in[14], h1[32], h2[32];
        for (int k = 0; k < 14; k++) in[k] = x[r * 14 + k];
        for (int o = 0; o < 32; o++) {
            float a = 0.f;
            for (int k = 0; k < 14; k++) a += W1[o * 14 + k] * in[k];
            h1[o] = fmaxf(a + b1[o], 0.f);
        }
        for (int o = 0; o < 32; o++) {
            float a = 0.f;
            for (int k = 0; k < 32; k++) a += W2[o * 32 + k] * h1[k];
            h2[o] = fmaxf(a + b2[o], 0.f);
        }
        uint32_t outw[4];
        float y[8];
        for (int o = 0; o < 6; o++) {
            float a = 0.f;
            for (int k = 0; k < 32; k++) a += W3[o * 32 + k] * h2[k];
            y[o] = a + b3[o];
        }
        y[6] = y[7] = 0.f;
        for (int e = 0; e < 4; e++) outw[e] = pack_h2(y[2 * e], y[2 * e + 1]);
        reinterpret_cast<uint4 *>(feat)[r] = make_uint4(outw[0], outw[1], outw[2], outw[3]);
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_prep(const sc_scene &scene, const sc_camera &cam, const sc_opts &opts, const Ws &ws,
                        sc_frame_stats *stats, cudaStream_t st)
{
    SC_LAUNCH(k_prep, 1, 1024, 0, st, scene, cam, opts, ws, stats);
    return cudaGetLastError();
}

cudaError_t launch_cull(const sc_scene &scene, const sc_camera &cam, const sc_opts &opts, const Ws &ws,
                        sc_survivor *out, int64_t cap, sc_frame_stats *stats, cudaStream_t st)
{
    SC_LAUNCH(k_chunk_map, (int)std::max<int64_t>(1, std::min<int64_t>((ws.max_chunks + 255) / 256, sm_count() * 8)),
              256, 0, st, ws.inst, scene.n_instances, ws.ctr, ws.chunk_inst);
    const int grid = sm_count() * SC_CULL_CPS;   // CTAs per SM (32 TMEM columns each)
    SC_LAUNCH(k_cull, grid, kCullThreads, 0, st, scene, cam, opts, ws, out, (long long)cap, stats);
    cudaError_t e = scan_excl(ws.chunk_cnt, ws.chunk_cnt, &ws.ctr->total_chunks, ws.max_chunks, ws.scan_part,
                              &ws.ctr->survivors, &stats->survivors, st);
    if (e != cudaSuccess) return e;
    SC_LAUNCH(k_compact, sm_count() * 16, 256, 0, st, ws.chunk_state, ws.chunk_cnt, ws.chunk_stage,
              &ws.ctr->total_chunks, &ws.ctr->survivors, out, (long long)cap, stats);
    return cudaGetLastError();
}

cudaError_t launch_vis_mlp(const sc_vis_weights *w, const float *x, int64_t n, float *logits, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    const int64_t tiles = (n + 127) / 128;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * 12);
    SC_LAUNCH(k_vis_forward, grid, 128, 0, st, w, x, n, logits);
    return cudaGetLastError();
}

cudaError_t launch_encode_features(const float *params, const float *x, int64_t n, uint16_t *feat,
                                   cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
    SC_LAUNCH(k_encode_features, grid, 256, 0, st, params, x, n, feat);
    return cudaGetLastError();
}

}  // namespace sc
