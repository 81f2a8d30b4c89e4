// Stage (c): instanced projection + SH colour + opacity, on survivors only.
//
// Compiled with -fmad=false.  Per survivor the kernel instantiates the
// Gaussian (B2: f64 -> f32, never stored), then follows the reference
// projection (sc/_kernels.py:35-133) operation by operation in float64, the
// radius clip and tile rectangle (sc/raster.py:289-316) and SH colour
// (sc/raster.py:198-226), and emits the 48-byte blend record, the depth sort
// key and the tile rectangle.
#include <algorithm>

#include "common.cuh"

namespace sc {

// real SH basis constants (sc/raster.py:30-37), f32: degrees >= 1 are evaluated in f32 (fp16 colours)
constexpr float kShC0 = 0.28209479177387814f;
constexpr float kShC1 = 0.4886025119029199f;
__constant__ float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                               -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f, 0.3731763325901154f,
                               -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};

__device__ __forceinline__ sc_survivor make_survivor(uint32_t inst, uint32_t gid)
{
    sc_survivor s;
    s.inst = inst;
    s.gid = gid;
    return s;
}


// sqrt.approx (rel. error < 2^-22): only where the result is widened by a margin far larger
__device__ __forceinline__ float sqrt_approx(float x)
{
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// rcp.approx (rel. error < 2^-23): the f32 conic only (tolerance-checked, never a decision)
__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// floor / ceil of an f64 value as int32, saturating (cvt.rmi / cvt.rpi clamp to the int range)
__device__ __forceinline__ int ifloor(double v) { return __double2int_rd(v); }
__device__ __forceinline__ int iceil(double v) { return __double2int_ru(v); }
__device__ __forceinline__ int iclamp(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// f32 dot product with explicit FMA (this TU is -fmad=false for the f64 paths)
__device__ __forceinline__ float fdot3(float a0, float a1, float a2, float b0, float b1, float b2)
{
    return fmaf(a0, b0, fmaf(a1, b1, a2 * b2));
}

// MODE kProjMixed: f32 covariance, exact f64 fallback inline (stage API);
// kProjFast: f32 only, ambiguous splats are appended to `list` (+ ctr->proj_deferred)
//            and projected afterwards by the exact kernel (frame path: keeps this
//            kernel small enough for 4 CTAs per SM);
// kProjExact: all-f64 reference path, over `list` when it is given.
// kProjFrame: kProjFast inside the frame path (keys written; no stage-API outputs, no
//            exact depth range: compile-time, not pointer tests)
enum { kProjMixed = 0, kProjFast = 1, kProjExact = 2, kProjFrame = 3 };

// frame-path kernel: 128-thread CTAs, 5 per SM (<= 102 registers: 96, no spills): 20 warps
// per SM; 256 x 2 (123 registers) gave 16, 128 x 6 (80 registers) spills (A/B: -1.3 % /
// +0.5 % frame).  The stage-API / exact instances keep their registers (no spills).
#ifndef SC_PROJ_CPS
#define SC_PROJ_CPS 5
#endif
#ifndef SC_PROJ_THREADS
#define SC_PROJ_THREADS 128
#endif
constexpr int kProjThreads = SC_PROJ_THREADS;
template <int MODE>
__global__ void __launch_bounds__(kProjThreads, MODE == kProjFrame ? SC_PROJ_CPS : 2) k_project(
    sc_scene scene, const sc_survivor *surv, const unsigned long long *n_dev, int64_t n_host, sc_camera cam,
    sc_opts opts, sc_splat *splats, sc_window *wins, double *depth64, ushort4 *rect, uint32_t *keys, uint2 *pv,
    double *dbg_f64, int32_t *dbg_rect, uint8_t *dbg_flags, sc_frame_stats *stats, Counters *ctr, uint32_t *list)
{
    // frame path: depth keys quantised over the instance spheres' depth range (k_prep)
    const double key_dmin = keys ? ctr->key_dmin : 0.0, key_scale = keys ? ctr->key_scale : 0.0;
    constexpr bool kDefer = MODE == kProjFast || MODE == kProjFrame;   // f32 only, ambiguous splats deferred
    if constexpr (MODE == kProjFrame) {
        depth64 = nullptr; rect = nullptr; dbg_f64 = nullptr; dbg_rect = nullptr; dbg_flags = nullptr;
    }
    const int64_t n_surv = n_dev ? min((int64_t)*n_dev, n_host) : n_host;
    const bool from_list = MODE == kProjExact && list != nullptr;
    const int64_t n = from_list ? (int64_t)ctr->proj_deferred : n_surv;
    const double lim_x = 1.3 * cam.tan_x, lim_y = 1.3 * cam.tan_y;
    const float lim_xf = (float)lim_x, lim_yf = (float)lim_y;
    const double focal = cam.focal;
    const int ts = opts.tile_size;
    const int tsh = (ts & (ts - 1)) == 0 ? __ffs(ts) - 1 : -1;   // log2 of a power-of-two tile size
    const int n_tx = (cam.width + ts - 1) / ts;
    const Band band = band_of(opts, cam.height, ts);
    unsigned long long n_passed = 0, n_skipped = 0, dmin_inv = 0, dmax_bits = 0, n_tentries = 0, n_exact = 0;
    const bool fast = kDefer || (MODE == kProjMixed && opts.exact_projection == 0);
    // camera rotation in f32 for the f32 covariance path (loop invariant)
    const float clip_f = opts.radius_clip > 0.0 ? (float)opts.radius_clip : 0.0f;
    const float pos_x = (float)cam.pos[0], pos_y = (float)cam.pos[1], pos_z = (float)cam.pos[2];
    const float r0 = (float)cam.rot[0], r1 = (float)cam.rot[1], r2 = (float)cam.rot[2], r3 = (float)cam.rot[3],
                r4 = (float)cam.rot[4], r5 = (float)cam.rot[5], r6 = (float)cam.rot[6], r7 = (float)cam.rot[7],
                r8 = (float)cam.rot[8];

    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // the survivor record is loaded one iteration ahead (the instance / Gaussian loads of an
    // iteration then start without waiting on it)
    int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    sc_survivor sv_next = make_survivor(0u, 0u);
    if (it < n) sv_next = surv[from_list ? (int64_t)list[it] : it];
    for (; it < n; it += stride) {
        const int64_t k = from_list ? (int64_t)list[it] : it;
        const sc_survivor sv = sv_next;
        if (it + stride < n) sv_next = surv[from_list ? (int64_t)list[it + stride] : it + stride];
        const sc_instance_rec &in = scene.instances[sv.inst];
        const sc_asset_rec &as = scene.assets[in.asset];
        const int64_t g = as.offset + sv.gid;
        const float4 mo = __ldg(reinterpret_cast<const float4 *>(scene.mean_opa) + g);
        const float4 q4 = __ldg(reinterpret_cast<const float4 *>(scene.quat) + g);
        const float4 ls4 = __ldg(reinterpret_cast<const float4 *>(scene.scale_smax) + g);

        // --- instancing (B2), exactly as the oracle's orc_instantiate ---
        const float3 mw = inst_mean(in, mo.x, mo.y, mo.z);
        // q' = q_i (x) q in f64 -> f32 (B2) for both paths: the instanced render must equal the
        // flattened one bit for bit, so q' is the same f32 value in either
        const float4 qw = inst_quat(in, q4);
        const float4 qf = qw;
        const float ls0 = __double2float_rn((double)ls4.x + in.ln_s);
        const float ls1 = __double2float_rn((double)ls4.y + in.ln_s);
        const float ls2 = __double2float_rn((double)ls4.z + in.ln_s);

        // --- projection (sc/_kernels.py:35-133) ---
        const double m0 = mw.x, m1 = mw.y, m2 = mw.z;
        double tx, ty, tz;
        cam_xyz(cam, m0, m1, m2, tx, ty, tz);
        bool valid = false;
        double mx = 0.0, my = 0.0, ca = 0.0, cb = 0.0, cc = 0.0, radius = 0.0, det = 0.0, cov_a = 0.0, cov_c = 0.0;
        // fast path (f32 end to end): half conic a / c, b, det and the conservative a, c of the support box
        float f_ha = 0.0f, f_b = 0.0f, f_hc = 0.0f, f_det = 0.0f, f_sa = 0.0f, f_sc = 0.0f;
        bool fast_done = false;
        if (tz > cam.near_) {
            const double txz = tx / tz, tyz = ty / tz;
            mx = focal * txz + (double)(cam.width - 1) / 2.0;
            my = focal * tyz + (double)(cam.height - 1) / 2.0;
            const double *R = cam.rot;
            if (fast) {
                // ---- f32 covariance / conic / eigenvalue with an error bound ----
                // Every product below is bounded in magnitude by the "absolute"
                // quadratic forms Ma = (sum |j0i| sqrt(g_ii))^2 (same for c, b), so the
                // accumulated f32 error of a, b, c is <= K eps (Ma + Mc + 2 Mb) (K
                // generous: ~40 dependent roundings, f32 exp, f32 quaternion product).
                // The radius is taken from f32 only when the whole interval of lambda
                // gives the same ceil(3 sqrt(lambda)); else the f64 path below runs.
                const float fz = (float)focal * rcp_approx((float)tz);   // <= 5 eps (K below has +8 for it)
                // (float) of the f64 clamp below == the f32 clamp of (float) txz (rounding is monotone)
                const float cx = fminf(fmaxf((float)txz, -lim_xf), lim_xf);
                const float cy = fminf(fmaxf((float)tyz, -lim_yf), lim_yf);
                const float j00 = fz * fmaf(-cx, r6, r0), j01 = fz * fmaf(-cx, r7, r1), j02 = fz * fmaf(-cx, r8, r2);
                const float j10 = fz * fmaf(-cy, r6, r3), j11 = fz * fmaf(-cy, r7, r4), j12 = fz * fmaf(-cy, r8, r5);
                const float qn = rsqrtf(fmaf(qf.x, qf.x, fdot3(qf.y, qf.z, qf.w, qf.y, qf.z, qf.w)));
                const float w = qf.x * qn, x = qf.y * qn, y = qf.z * qn, z = qf.w * qn;
                const float q00 = 1.0f - 2.0f * (y * y + z * z), q01 = 2.0f * (x * y - w * z), q02 = 2.0f * (x * z + w * y);
                const float q10 = 2.0f * (x * y + w * z), q11 = 1.0f - 2.0f * (x * x + z * z), q12 = 2.0f * (y * z - w * x);
                const float q20 = 2.0f * (x * z - w * y), q21 = 2.0f * (y * z + w * x), q22 = 1.0f - 2.0f * (x * x + y * y);
                const float s0 = __expf(2.0f * ls0), s1 = __expf(2.0f * ls1), s2 = __expf(2.0f * ls2);   // 2 ulp: inside K
                const float g00 = fdot3(q00 * q00, q01 * q01, q02 * q02, s0, s1, s2);
                const float g01 = fdot3(q00 * q10, q01 * q11, q02 * q12, s0, s1, s2);
                const float g02 = fdot3(q00 * q20, q01 * q21, q02 * q22, s0, s1, s2);
                const float g11 = fdot3(q10 * q10, q11 * q11, q12 * q12, s0, s1, s2);
                const float g12 = fdot3(q10 * q20, q11 * q21, q12 * q22, s0, s1, s2);
                const float g22 = fdot3(q20 * q20, q21 * q21, q22 * q22, s0, s1, s2);
                const float u0 = fdot3(j00, j01, j02, g00, g01, g02);
                const float u1 = fdot3(j00, j01, j02, g01, g11, g12);
                const float u2 = fdot3(j00, j01, j02, g02, g12, g22);
                const float v0 = fdot3(j10, j11, j12, g00, g01, g02);
                const float v1 = fdot3(j10, j11, j12, g01, g11, g12);
                const float v2 = fdot3(j10, j11, j12, g02, g12, g22);
                const float dil = (float)opts.dilation;
                const float fa = fdot3(u0, u1, u2, j00, j01, j02) + dil;
                const float fb = fdot3(u0, u1, u2, j10, j11, j12);
                const float fc = fdot3(v0, v1, v2, j10, j11, j12) + dil;
                // (na + nc)^2 with na = sum |j0i| sqrt(g_ii) (nc likewise) is bounded without a
                // square root by Cauchy-Schwarz: <= 2 tr(Sigma) (|J0|^2 + |J1|^2), tr(Sigma) =
                // s0 + s1 + s2 (rotation invariant; 1e-3 slack for the f32 rotation's norm)
                const float jn = fdot3(j00, j01, j02, j00, j01, j02) + fdot3(j10, j11, j12, j10, j11, j12);
                const float nn = 2.002f * (s0 + s1 + s2) * jn;
                constexpr float kEps = 5.9604645e-08f, K = 72.0f;
                const float err = K * kEps * nn + 4.0f * kEps * fabsf(dil);
                const float hd = 0.5f * (fa - fc);
                // sqrt.approx (rel. error < 2^-22 = 4 eps) stays inside the 16 eps slack of lo / hi
                const float lam = 0.5f * (fa + fc) + sqrt_approx(fmaf(hd, hd, fb * fb));
                const float lo = fmaxf(lam * (1.0f - 16.0f * kEps) - 2.0f * err, 0.0f);
                const float hi = lam * (1.0f + 16.0f * kEps) + 2.0f * err;
                // radius = ceil(3 sqrt(lambda)) is the same integer rc for every lambda in [lo, hi] iff
                // (rc - 1)^2 < 9 lo and 9 hi <= rc^2 (squares exact in f32 below 4096; 9 x rounded
                // with margin): one square root instead of one per interval end
                const float rc = ceilf(3.0f * sqrt_approx(lam));   // any rc: the test below validates it
                const bool r_ok = rc >= 1.0f && rc <= 4000.0f && (rc - 1.0f) * (rc - 1.0f) < 9.0f * lo * (1.0f - 8.0f * kEps) &&
                                  9.0f * hi * (1.0f + 8.0f * kEps) <= rc * rc;
                const float rlo = r_ok ? rc : 0.0f, rhi = r_ok ? rc : -1.0f;
                // det = a c - b^2 in f32 with one FMA-exact square (Kahan): |error| <= 2 eps |det|,
                // added to the bound below together with the f32 rounding of radius_clip
                const float bb = fb * fb;
                const float fdet = fmaf(fa, fc, -bb) - fmaf(fb, fb, -bb);
                const float det_err = 4.0f * err * (fa + fc + 2.0f * err) + 4.0f * kEps * fabsf(fdet) +
                                      2.0f * kEps * clip_f + 1e-30f;
                const bool clip_ok = !(clip_f > 0.0f) || fabsf(fdet - clip_f) > det_err;
                if (rlo == rhi && fdet - det_err > 1e-12f && clip_ok) {
                    fast_done = true;
                    radius = (double)rlo;
                    f_det = fdet;
                    const float inv = rcp_approx(fdet);   // fdet > 1e-12: a normal positive number
                    f_ha = 0.5f * (fc * inv);
                    f_b = -fb * inv;
                    f_hc = 0.5f * (fa * inv);
                    valid = rlo > 0.0f;
                    if (valid && clip_f > 0.0f && fdet < clip_f) valid = false;   // det == fdet (dbg only)
                    // support box from the conservative a, c (times 2 L later)
                    f_sa = fa + err;
                    f_sc = fc + err;
                }
            }
            if constexpr (kDefer) {
                if (!fast_done) {   // ambiguous: the exact kernel projects this splat afterwards
                    list[atomicAdd(&ctr->proj_deferred, 1ull)] = (uint32_t)k;
                    n_exact++;
                    continue;
                }
            }
            if (!kDefer && !fast_done) {
                if (fast) n_exact++;
                const double fz = focal / tz;
                const double ctxz = fmin(fmax(txz, -lim_x), lim_x);
                const double ctyz = fmin(fmax(tyz, -lim_y), lim_y);
                const double j00 = fz * R[0] - fz * ctxz * R[6];
                const double j01 = fz * R[1] - fz * ctxz * R[7];
                const double j02 = fz * R[2] - fz * ctxz * R[8];
                const double j10 = fz * R[3] - fz * ctyz * R[6];
                const double j11 = fz * R[4] - fz * ctyz * R[7];
                const double j12 = fz * R[5] - fz * ctyz * R[8];

                const double q0 = qw.x, q1 = qw.y, q2 = qw.z, q3 = qw.w;
                const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
                const double w = q0 / qn, x = q1 / qn, y = q2 / qn, z = q3 / qn;
                const double r00 = 1.0 - 2.0 * (y * y + z * z);
                const double r01 = 2.0 * (x * y - w * z);
                const double r02 = 2.0 * (x * z + w * y);
                const double r10 = 2.0 * (x * y + w * z);
                const double r11 = 1.0 - 2.0 * (x * x + z * z);
                const double r12 = 2.0 * (y * z - w * x);
                const double r20 = 2.0 * (x * z - w * y);
                const double r21 = 2.0 * (y * z + w * x);
                const double r22 = 1.0 - 2.0 * (x * x + y * y);
                const double s0 = exp(2.0 * (double)ls0);
                const double s1 = exp(2.0 * (double)ls1);
                const double s2 = exp(2.0 * (double)ls2);
                const double g00 = r00 * r00 * s0 + r01 * r01 * s1 + r02 * r02 * s2;
                const double g01 = r00 * r10 * s0 + r01 * r11 * s1 + r02 * r12 * s2;
                const double g02 = r00 * r20 * s0 + r01 * r21 * s1 + r02 * r22 * s2;
                const double g11 = r10 * r10 * s0 + r11 * r11 * s1 + r12 * r12 * s2;
                const double g12 = r10 * r20 * s0 + r11 * r21 * s1 + r12 * r22 * s2;
                const double g22 = r20 * r20 * s0 + r21 * r21 * s1 + r22 * r22 * s2;
                const double u0 = j00 * g00 + j01 * g01 + j02 * g02;
                const double u1 = j00 * g01 + j01 * g11 + j02 * g12;
                const double u2 = j00 * g02 + j01 * g12 + j02 * g22;
                const double v0 = j10 * g00 + j11 * g01 + j12 * g02;
                const double v1 = j10 * g01 + j11 * g11 + j12 * g12;
                const double v2 = j10 * g02 + j11 * g12 + j12 * g22;
                const double a = u0 * j00 + u1 * j01 + u2 * j02 + opts.dilation;
                const double b = u0 * j10 + u1 * j11 + u2 * j12;
                const double c = v0 * j10 + v1 * j11 + v2 * j12 + opts.dilation;
                cov_a = a;
                cov_c = c;
                det = a * c - b * b;
                if (det <= 1e-12) {
                    n_skipped++;
                } else {
                    ca = c / det;
                    cb = -b / det;
                    cc = a / det;
                    const double mid = 0.5 * (a + c);
                    const double disc = mid * mid - det;
                    const double lam = mid + sqrt(disc > 0.0 ? disc : 0.0);
                    radius = ceil(3.0 * sqrt(lam));
                    valid = radius > 0.0;
                    if (valid && opts.radius_clip > 0.0 && det < opts.radius_clip) valid = false;
                }
            }
        }
        // --- tile rectangle (sc/raster.py:307-314) ---
        // power-of-two tile sizes: floor((m -+ r) / ts) == floor(m -+ r) >> log2(ts) (the
        // f64 difference is rounded once either way, / 2^k is exact, and floor(floor(x) /
        // 2^k) == floor(x / 2^k)); other sizes divide in f64 exactly as the reference.
        // The int conversions saturate, which the clamps below absorb.
        int tx0 = 0, tx1 = 0, ty0 = 0, ty1 = 0;
        int fx0 = 0, fx1 = 0, fy0 = 0, fy1 = 0;   // floor(m - r), floor(m + r)
        bool passed = false;
        if (valid) {
            const double vx0 = mx - radius, vx1 = mx + radius, vy0 = my - radius, vy1 = my + radius;
            fx0 = ifloor(vx0);
            fx1 = ifloor(vx1);
            fy0 = ifloor(vy0);
            fy1 = ifloor(vy1);
            int qx0, qx1, qy0, qy1;
            if (tsh >= 0) {
                qx0 = fx0 >> tsh; qx1 = fx1 >> tsh; qy0 = fy0 >> tsh; qy1 = fy1 >> tsh;
            } else {
                const double dts = (double)ts;
                qx0 = ifloor(vx0 / dts); qx1 = ifloor(vx1 / dts); qy0 = ifloor(vy0 / dts); qy1 = ifloor(vy1 / dts);
            }
            tx0 = iclamp(qx0, 0, n_tx);
            tx1 = iclamp(min(qx1, 0x7FFFFFFE) + 1, 0, n_tx);
            // tile rows clamp to the band (the whole image: [0, n_ty))
            ty0 = iclamp(qy0, band.t0, band.t1);
            ty1 = iclamp(min(qy1, 0x7FFFFFFE) + 1, band.t0, band.t1);
            passed = tx1 > tx0 && ty1 > ty0;
        }
        n_passed += passed;
        if (passed) {
            n_tentries += (unsigned long long)((tx1 - tx0) * (ty1 - ty0));   // reference tile entries
            if constexpr (MODE != kProjFrame) {   // the stage API's key range (k_depth_keys)
                const unsigned long long bits = (unsigned long long)__double_as_longlong(tz);
                dmin_inv = max(dmin_inv, ~bits);
                dmax_bits = max(dmax_bits, bits);
            }
        }

        // --- colour (sc/raster.py:198-226) and opacity (sc/asset.py:44-51) ---
        // Per-gaussian, view-independent parts come precomputed (DeviceScene, f64 like the
        // reference, rounded once): p_min = ln(1/255) - ln(sigmoid(logit)) (+inf when the
        // reference skips the splat, opacity < 1/255) and the degree-0 colour in fp16.
        // Higher degrees are evaluated here in f32 (the colour is stored as fp16).
        const float4 ap = __ldg(reinterpret_cast<const float4 *>(scene.appear) + g);
        const float p_min = ap.x;
        const bool skip = !(p_min < __int_as_float(0x7f800000));
        int deg = as.sh_degree;
        if (opts.sh_degree_eval >= 0 && opts.sh_degree_eval < deg) deg = opts.sh_degree_eval;
        sc_splat sp;
        if (deg == 0) {
            const uint32_t rg = __float_as_uint(ap.y), bz = __float_as_uint(ap.z);
            sp.rgb[0] = (uint16_t)(rg & 0xFFFFu);
            sp.rgb[1] = (uint16_t)(rg >> 16);
            sp.rgb[2] = (uint16_t)(bz & 0xFFFFu);
        } else {
            const float *shp = scene.sh + g * (int64_t)scene.sh_stride;
            float dx = mw.x - pos_x, dy = mw.y - pos_y, dz = mw.z - pos_z;
            const float rn = rsqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
            dx *= rn;
            dy *= rn;
            dz *= rn;
            const float C0 = kShC0, C1 = kShC1;
            float col[3];
            for (int ch = 0; ch < 3; ch++) {
                col[ch] = C0 * __ldg(shp + ch) - C1 * dy * __ldg(shp + 3 + ch) + C1 * dz * __ldg(shp + 6 + ch) -
                          C1 * dx * __ldg(shp + 9 + ch);
            }
            if (deg >= 2) {
                const float xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yz = dy * dz, xz = dx * dz;
                for (int ch = 0; ch < 3; ch++) {
                    const float *c = shp + ch;
                    col[ch] += kShC2[0] * xy * __ldg(c + 12) + kShC2[1] * yz * __ldg(c + 15) +
                               kShC2[2] * (2.0f * zz - xx - yy) * __ldg(c + 18) +
                               kShC2[3] * xz * __ldg(c + 21) + kShC2[4] * (xx - yy) * __ldg(c + 24);
                }
                if (deg >= 3) {
                    for (int ch = 0; ch < 3; ch++) {
                        const float *c = shp + ch;
                        col[ch] += kShC3[0] * dy * (3.0f * xx - yy) * __ldg(c + 27) +
                                   kShC3[1] * xy * dz * __ldg(c + 30) +
                                   kShC3[2] * dy * (4.0f * zz - xx - yy) * __ldg(c + 33) +
                                   kShC3[3] * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy) * __ldg(c + 36) +
                                   kShC3[4] * dx * (4.0f * zz - xx - yy) * __ldg(c + 39) +
                                   kShC3[5] * dz * (xx - yy) * __ldg(c + 42) +
                                   kShC3[6] * dx * (xx - 3.0f * yy) * __ldg(c + 45);
                    }
                }
            }
            for (int ch = 0; ch < 3; ch++)
                sp.rgb[ch] = __half_as_ushort(__float2half_rn(fminf(fmaxf(col[ch] + 0.5f, 0.0f), 1.0f)));
        }
        sp.mx = (float)mx;
        sp.my = (float)my;
        if (fast_done) {
            sp.half_a = f_ha;
            sp.b = f_b;
            sp.half_c = f_hc;
        } else {
            sp.half_a = (float)(0.5 * ca);
            sp.b = (float)cb;
            sp.half_c = (float)(0.5 * cc);
        }
        sp.p_min = p_min;
        sp.reserved = 0;
        sc_window win;
        if (passed && !skip) {
            // reference pixel window (sc/_kernels.py:224-227), intersected with the
            // bounding box of the alpha >= 1/255 support {1/2 d^T cov^-1 d <= L},
            // L = log(op) - log(1/255) = -p_min: |dx| <= sqrt(2 L cov_xx).  Pixels
            // outside the box fail the reference's `power < p_min` test, so the image
            // is unchanged; the box is widened for safety.  Also clipped to the
            // splat's tile rectangle in pixels: the reference only composites a splat
            // inside tiles whose list holds it, and its window can reach one pixel
            // past the rect (A8 step 3).  Integer form of max(floor(m - r), ceil(m -
            // e), ts t0) / min(floor(m + r) + 1, floor(m + e), ts t1 - 1), clamped to
            // the int16 window range [-1, 32767].
            int bx0, bx1, by0, by1;
            if (fast_done) {
                // f32: a, c widened by their error bound, then 1e-4 relative + 1e-2 px, plus the
                // f32 rounding of m and of the sums (1e-3 px + 2.4e-7 relative)
                const float l2 = -2.0f * p_min;
                const float ex = fmaf(sqrt_approx(l2 * f_sa), 1.0001f, 0.01f);
                const float ey = fmaf(sqrt_approx(l2 * f_sc), 1.0001f, 0.01f);
                const float mxf = sp.mx, myf = sp.my;
                const float gx = ex + 1e-3f + 2.4e-7f * (fabsf(mxf) + ex);
                const float gy = ey + 1e-3f + 2.4e-7f * (fabsf(myf) + ey);
                bx0 = __float2int_ru(mxf - gx);
                bx1 = __float2int_rd(mxf + gx);
                by0 = __float2int_ru(myf - gy);
                by1 = __float2int_rd(myf + gy);
            } else {
                const double L = -(double)p_min;
                const double ex = sqrt(2.0 * L * cov_a) * (1.0 + 1e-5) + 1e-3;
                const double ey = sqrt(2.0 * L * cov_c) * (1.0 + 1e-5) + 1e-3;
                bx0 = iceil(mx - ex);
                bx1 = ifloor(mx + ex);
                by0 = iceil(my - ey);
                by1 = ifloor(my + ey);
            }
            win.x0 = (int16_t)iclamp(max(max(fx0, bx0), ts * tx0), -1, 32767);
            win.x1 = (int16_t)iclamp(min(min(min(fx1, 0x7FFFFFFE) + 1, bx1), ts * tx1 - 1), -1, 32767);
            win.y0 = (int16_t)iclamp(max(max(fy0, by0), ts * ty0), -1, 32767);
            win.y1 = (int16_t)iclamp(min(min(min(fy1, 0x7FFFFFFE) + 1, by1), ts * ty1 - 1), -1, 32767);
        } else {   // never composited
            win.x0 = 1;
            win.x1 = 0;
            win.y0 = 1;
            win.y1 = 0;
        }
        splats[k] = sp;
        const uint32_t packed = passed ? pack_window(win.x0, win.x1, win.y0, win.y1, cam.width, cam.height) : kWinEmpty;
        if (!keys || packed == kWinEscape) wins[k] = win;   // frame path: only escapes are read back
        if (depth64) depth64[k] = passed ? tz : -1.0;   // stage API: sort keys are quantised in k_depth_keys
        if (keys) {
            // monotone non-decreasing in tz (clamped subtraction, positive scale, floor): equal keys are
            // re-ordered by (tz, index) in the tie-fix; non-passed splats sink to the end
            constexpr double kTop = 4294967040.0;
            // (cvt.rmi.u32.f64 clamps to [0, 2^32 - 1]: floor(max(x, 0)) in one conversion)
            keys[k] = passed ? min(__double2uint_rd((tz - key_dmin) * key_scale), (uint32_t)kTop) : 0xFFFFFFFFu;
            reinterpret_cast<uint32_t *>(pv)[k] = packed;   // the first depth pass adds the index (= k)
        }
        if (rect) rect[k] = make_ushort4((unsigned short)tx0, (unsigned short)tx1, (unsigned short)ty0, (unsigned short)ty1);
        if (dbg_f64) {
            double *d = dbg_f64 + 8 * k;
            if (fast_done) {   // the f32 conic (0.5 a and 0.5 c are exact halvings) and det
                ca = 2.0 * (double)f_ha;
                cb = (double)f_b;
                cc = 2.0 * (double)f_hc;
                det = (double)f_det;
            }
            d[0] = mx; d[1] = my; d[2] = ca; d[3] = cb; d[4] = cc; d[5] = tz; d[6] = radius; d[7] = det;
        }
        if (dbg_rect) {
            dbg_rect[4 * k] = tx0; dbg_rect[4 * k + 1] = tx1; dbg_rect[4 * k + 2] = ty0; dbg_rect[4 * k + 3] = ty1;
        }
        if (dbg_flags) dbg_flags[k] = (uint8_t)((valid ? 1 : 0) | (passed ? 2 : 0));
    }
    for (int o = 16; o > 0; o >>= 1) {
        n_passed += __shfl_down_sync(0xffffffffu, n_passed, o);
        n_skipped += __shfl_down_sync(0xffffffffu, n_skipped, o);
        n_tentries += __shfl_down_sync(0xffffffffu, n_tentries, o);
        n_exact += __shfl_down_sync(0xffffffffu, n_exact, o);
        dmin_inv = max(dmin_inv, __shfl_down_sync(0xffffffffu, dmin_inv, o));
        dmax_bits = max(dmax_bits, __shfl_down_sync(0xffffffffu, dmax_bits, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (n_passed) {
            atomicAdd((unsigned long long *)&stats->passed, n_passed);
            if (ctr) {
                atomicAdd(&ctr->passed, n_passed);
                atomicMax(&ctr->dmin_inv, dmin_inv);
                atomicMax(&ctr->dmax, dmax_bits);
            }
        }
        if (n_skipped) atomicAdd((unsigned long long *)&stats->skipped, n_skipped);
        if (n_tentries) atomicAdd((unsigned long long *)&stats->entries, n_tentries);
        if (fast && n_exact) atomicAdd((unsigned long long *)&stats->exact_fallbacks, n_exact);
    }
}

cudaError_t launch_project(const sc_scene &scene, const sc_survivor *surv, const unsigned long long *n_dev,
                           int64_t n_max, const sc_camera &cam, const sc_opts &opts, sc_splat *splats,
                           sc_window *wins, double *depth64, ushort4 *rect, uint32_t *keys, uint2 *pv,
                           double *dbg_f64, int32_t *dbg_rect, uint8_t *dbg_flags, sc_frame_stats *stats,
                           Counters *ctr, uint32_t *defer_list, cudaStream_t st)
{
    if (n_max <= 0) return cudaSuccess;
    const int nsm = sm_count();
#ifndef SC_PROJ_GRID
#define SC_PROJ_GRID SC_PROJ_CPS   // one wave of resident CTAs: no partial last wave
#endif
    const int64_t blocks = std::min<int64_t>((n_max + kProjThreads - 1) / kProjThreads, (int64_t)nsm * SC_PROJ_GRID);
    if (opts.exact_projection) {
        SC_LAUNCH(k_project<kProjExact>, (int)blocks, kProjThreads, 0, st, scene, surv, n_dev, n_max, cam, opts, splats, wins,
                  depth64, rect, keys, pv, dbg_f64, dbg_rect, dbg_flags, stats, ctr, nullptr);
    } else if (defer_list && ctr) {   // lean f32 kernel, then the exact kernel over the deferred splats
        if (keys && !depth64 && !rect && !dbg_f64 && !dbg_rect && !dbg_flags)   // the frame path
            SC_LAUNCH(k_project<kProjFrame>, (int)blocks, kProjThreads, 0, st, scene, surv, n_dev, n_max, cam, opts, splats,
                      wins, depth64, rect, keys, pv, dbg_f64, dbg_rect, dbg_flags, stats, ctr, defer_list);
        else
            SC_LAUNCH(k_project<kProjFast>, (int)blocks, kProjThreads, 0, st, scene, surv, n_dev, n_max, cam, opts, splats,
                      wins, depth64, rect, keys, pv, dbg_f64, dbg_rect, dbg_flags, stats, ctr, defer_list);
        SC_LAUNCH(k_project<kProjExact>, nsm, kProjThreads, 0, st, scene, surv, n_dev, n_max, cam, opts, splats, wins, depth64,
                  rect, keys, pv, dbg_f64, dbg_rect, dbg_flags, stats, ctr, defer_list);
    } else {
        SC_LAUNCH(k_project<kProjMixed>, (int)blocks, kProjThreads, 0, st, scene, surv, n_dev, n_max, cam, opts, splats, wins,
                  depth64, rect, keys, pv, dbg_f64, dbg_rect, dbg_flags, stats, ctr, nullptr);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// tie-fix: runs of equal depth keys -> (f64 depth, survivor index) order, the
// reference's argsort(kind="stable") order (sc/raster.py:319).  The depth is
// read from depth64 (stage API) or recomputed from the survivor exactly as the
// projection computes it (frame path; this TU is -fmad=false).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double tie_depth(const sc_scene &scene, const sc_survivor *surv, const sc_camera &cam,
                                            const double *depth64, uint32_t idx)
{
    if (depth64) return depth64[idx];
    const sc_survivor sv = surv[idx];
    const sc_instance_rec &in = scene.instances[sv.inst];
    const int64_t g = scene.assets[in.asset].offset + sv.gid;
    const float4 mo = __ldg(reinterpret_cast<const float4 *>(scene.mean_opa) + g);
    const float3 mw = inst_mean(in, mo.x, mo.y, mo.z);
    double tx, ty, tz;
    cam_xyz(cam, mw.x, mw.y, mw.z, tx, ty, tz);
    return tz;
}

// pass 1: heads of runs of >= 2 equal keys -> run_list (order irrelevant).
// A thread scans 8 consecutive keys; one global atomic per 2048-key CTA chunk.
__global__ void __launch_bounds__(256) k_tie_heads(const uint32_t *keys, const unsigned long long *n_dev,
                                                   int64_t n_host, uint32_t *run_list, Counters *ctr)
{
    __shared__ uint32_t s_warp[8], s_base;
    const int64_t n = n_dev ? min((int64_t)*n_dev, n_host) : n_host;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t cbase = blockIdx.x * 2048ll; cbase < n; cbase += (int64_t)gridDim.x * 2048) {
        const int64_t i0 = cbase + 8 * threadIdx.x;
        uint32_t kv[10];   // keys i0 - 1 .. i0 + 8
        uint32_t heads = 0;
        if (i0 < n) {
            if (i0 + 8 <= n && (i0 & 3) == 0) {
                const uint4 a = __ldg(reinterpret_cast<const uint4 *>(keys + i0));
                const uint4 b = __ldg(reinterpret_cast<const uint4 *>(keys + i0) + 1);
                kv[1] = a.x; kv[2] = a.y; kv[3] = a.z; kv[4] = a.w; kv[5] = b.x; kv[6] = b.y; kv[7] = b.z; kv[8] = b.w;
            } else {
#pragma unroll
                for (int j = 0; j < 8; j++) kv[j + 1] = i0 + j < n ? keys[i0 + j] : 0u;
            }
            kv[0] = i0 > 0 ? keys[i0 - 1] : ~kv[1];
            kv[9] = i0 + 8 < n ? keys[i0 + 8] : 0u;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int64_t i = i0 + j;
                const bool h = i + 1 < n && kv[j] != kv[j + 1] && kv[j + 1] == kv[j + 2];
                heads |= (uint32_t)h << j;
            }
        }
        uint32_t c = __popc(heads), x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int w = 0; w < 8; w++) {
                const uint32_t ww = s_warp[w];
                s_warp[w] = t;
                t += ww;
            }
            s_base = t ? (uint32_t)atomicAdd(&ctr->tie_runs, (unsigned long long)t) : 0u;
        }
        __syncthreads();
        uint32_t slot = s_base + s_warp[wid] + x - c;
        while (heads) {
            const int j = __ffs(heads) - 1;
            heads &= heads - 1;
            run_list[slot++] = (uint32_t)(i0 + j);
        }
        __syncthreads();
    }
}

// pass 2: one thread per run, insertion sort on (depth, index); runs of up to
// kTieRegs elements have their depths computed independently (ILP)
constexpr int kTieRegs = 8;
__global__ void k_tie_runs(sc_scene scene, const sc_survivor *surv, sc_camera cam, const uint32_t *keys, uint2 *pv,
                           const double *depth64, const unsigned long long *n_dev, int64_t n_host,
                           const uint32_t *run_list, uint32_t *long_list, Counters *ctr, sc_frame_stats *stats)
{
    const int64_t n = n_dev ? min((int64_t)*n_dev, n_host) : n_host;
    const int64_t runs = (int64_t)ctr->tie_runs;
    unsigned long long longest = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < runs; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = run_list[r];
        const uint32_t key = keys[i];
        if (i + kTieRegs < n && keys[i + kTieRegs] == key) {   // longer than kTieRegs: one CTA per run
            long_list[atomicAdd(&ctr->tie_long, 1ull)] = (uint32_t)i;
            continue;
        }
        int64_t e = i + 1;
        while (e < n && keys[e] == key) e++;
        const int len = (int)(e - i);
        longest = max(longest, (unsigned long long)len);
        {
            uint2 v[kTieRegs];
            double d[kTieRegs];
#pragma unroll
            for (int q = 0; q < kTieRegs; q++)
                if (q < len) v[q] = pv[i + q];
#pragma unroll
            for (int q = 0; q < kTieRegs; q++)
                if (q < len) d[q] = tie_depth(scene, surv, cam, depth64, v[q].x);
#pragma unroll
            for (int a = 1; a < kTieRegs; a++) {
                if (a < len) {
#pragma unroll
                    for (int b = a; b > 0; b--) {   // bubble element a down (stable)
                        const bool sw = d[b] < d[b - 1] || (d[b] == d[b - 1] && v[b].x < v[b - 1].x);
                        if (sw) {
                            const double td = d[b]; d[b] = d[b - 1]; d[b - 1] = td;
                            const uint2 tv = v[b]; v[b] = v[b - 1]; v[b - 1] = tv;
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kTieRegs; q++)
                if (q < len) pv[i + q] = v[q];
        }
    }
    for (int o = 16; o > 0; o >>= 1) longest = max(longest, __shfl_down_sync(0xffffffffu, longest, o));
    if ((threadIdx.x & 31) == 0 && longest) atomicMax((unsigned long long *)&stats->max_tie_run, longest);
}

// pass 3: runs longer than kTieRegs, one CTA each: depths computed in parallel;
// runs already in (depth, index) order (e.g. a planar asset facing the camera:
// all depths equal) are left alone, others up to kTieSmem elements are
// bitonic-sorted in shared memory; longer ones are sorted by a CTA-wide
// ascending-only bitonic network (mirror first step per merge size, so the
// virtual +inf padding past the run never moves): merge steps with partner
// distance >= kTieSmem run in global memory over the run's own slice of the
// depth-sort ping-pong buffer (f64 depths, free after the depth sort), the
// shorter ones chunk by chunk in shared memory.
constexpr int kTieSmem = 2048;

__device__ __forceinline__ bool tie_less(double da, uint32_t ia, double db, uint32_t ib)
{
    return da < db || (da == db && ia < ib);
}

// one compare-exchange of positions lo < hi (min to lo) in global memory
__device__ __forceinline__ void tie_ce_global(double *d, uint2 *v, int64_t lo, int64_t hi)
{
    const double dl = d[lo], dh = d[hi];
    const uint2 vl = v[lo], vh = v[hi];
    if (tie_less(dh, vh.x, dl, vl.x)) {
        d[lo] = dh; d[hi] = dl;
        v[lo] = vh; v[hi] = vl;
    }
}

__global__ void __launch_bounds__(256) k_tie_long(sc_scene scene, const sc_survivor *surv, sc_camera cam,
                                                  const uint32_t *keys, uint2 *pv, const double *depth64,
                                                  const unsigned long long *n_dev, int64_t n_host,
                                                  const uint32_t *long_list, const Counters *ctr, sc_frame_stats *stats,
                                                  double *scratch)
{
    __shared__ double s_d[kTieSmem];
    __shared__ uint2 s_v[kTieSmem];
    __shared__ long long s_end;
    __shared__ int s_unsorted;
    const int64_t n = n_dev ? min((int64_t)*n_dev, n_host) : n_host;
    const int64_t runs = (int64_t)ctr->tie_long;
    const int tid = threadIdx.x;
    for (int64_t r = blockIdx.x; r < runs; r += gridDim.x) {
        const int64_t i = long_list[r];
        const uint32_t key = keys[i];
        // run end: probe 256 positions per round
        if (tid == 0) {
            s_end = n;
            s_unsorted = 0;
        }
        __syncthreads();
        for (int64_t base = i + 1;; base += 256) {
            const int64_t q = base + tid;
            const bool stop = q >= n || keys[q] != key;
            if (stop) atomicMin(&s_end, (long long)q);
            if (__syncthreads_or(stop)) break;
        }
        const int64_t e = s_end;
        const int64_t len = e - i;
        // already ordered? (the run is in index order: ordered iff depths are non-decreasing)
        for (int64_t a = i + 1 + tid; a < e; a += 256) {
            const double d0 = tie_depth(scene, surv, cam, depth64, pv[a - 1].x);
            const double d1 = tie_depth(scene, surv, cam, depth64, pv[a].x);
            if (d1 < d0) s_unsorted = 1;
        }
        __syncthreads();
        if (tid == 0) atomicMax((unsigned long long *)&stats->max_tie_run, (unsigned long long)len);
        if (!s_unsorted) {
            __syncthreads();
            continue;
        }
        if (len <= kTieSmem) {
            int p2 = 1;
            while (p2 < len) p2 <<= 1;
            for (int a = tid; a < p2; a += 256) {
                if (a < len) {
                    s_v[a] = pv[i + a];
                    s_d[a] = tie_depth(scene, surv, cam, depth64, s_v[a].x);
                } else {
                    s_v[a] = make_uint2(0xFFFFFFFFu, 0u);
                    s_d[a] = INFINITY;
                }
            }
            __syncthreads();
            for (int k = 2; k <= p2; k <<= 1)
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    for (int a = tid; a < p2; a += 256) {
                        const int b = a ^ jj;
                        if (b > a) {
                            const bool up = (a & k) == 0;
                            const bool gt = s_d[a] > s_d[b] || (s_d[a] == s_d[b] && s_v[a].x > s_v[b].x);
                            if (gt == up) {
                                const double td = s_d[a]; s_d[a] = s_d[b]; s_d[b] = td;
                                const uint2 tv = s_v[a]; s_v[a] = s_v[b]; s_v[b] = tv;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int a = tid; a < len; a += 256) pv[i + a] = s_v[a];
        } else {
            double *gd = scratch + i;   // this run's slice: runs are disjoint
            uint2 *gv = pv + i;
            for (int64_t a = tid; a < len; a += 256) gd[a] = tie_depth(scene, surv, cam, depth64, gv[a].x);
            __syncthreads();
            int64_t p2 = 1;
            while (p2 < len) p2 <<= 1;
            // chunk-local steps (partner distance < kTieSmem) of merge size k in shared memory;
            // kfull: the whole network up to merge size kTieSmem (first phase)
            auto smem_steps = [&](int64_t k, bool kfull) {
                for (int64_t c0 = 0; c0 < len; c0 += kTieSmem) {
                    const int cl = (int)min((int64_t)kTieSmem, len - c0);
                    for (int a = tid; a < kTieSmem; a += 256) {
                        s_d[a] = a < cl ? gd[c0 + a] : INFINITY;
                        s_v[a] = a < cl ? gv[c0 + a] : make_uint2(0xFFFFFFFFu, 0u);
                    }
                    __syncthreads();
                    const int k0 = kfull ? 2 : (int)kTieSmem;   // merge sizes handled here
                    for (int kk = k0; kk <= (kfull ? kTieSmem : kTieSmem); kk <<= 1) {
                        const bool mirror_here = kfull;
                        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                            if (!kfull && jj >= kTieSmem) continue;
                            for (int a = tid; a < kTieSmem; a += 256) {
                                int b;
                                if (mirror_here && jj == (kk >> 1)) b = (a & ~(kk - 1)) + (kk - 1 - (a & (kk - 1)));
                                else b = a ^ jj;
                                if (b > a && tie_less(s_d[b], s_v[b].x, s_d[a], s_v[a].x)) {
                                    const double td = s_d[a]; s_d[a] = s_d[b]; s_d[b] = td;
                                    const uint2 tv = s_v[a]; s_v[a] = s_v[b]; s_v[b] = tv;
                                }
                            }
                            __syncthreads();
                        }
                        if (!kfull) break;
                    }
                    for (int a = tid; a < cl; a += 256) {
                        gd[c0 + a] = s_d[a];
                        gv[c0 + a] = s_v[a];
                    }
                    __syncthreads();
                }
                (void)k;
            };
            smem_steps(kTieSmem, true);   // every chunk sorted
            for (int64_t k = 2 * kTieSmem; k <= p2; k <<= 1) {
                for (int64_t jj = k >> 1; jj >= kTieSmem; jj >>= 1) {
                    const bool mirror = jj == (k >> 1);
                    for (int64_t a = tid; a < p2; a += 256) {
                        const int64_t b = mirror ? (a & ~(k - 1)) + (k - 1 - (a & (k - 1))) : (a ^ jj);
                        if (b > a && b < len) tie_ce_global(gd, gv, a, b);
                    }
                    __syncthreads();
                }
                smem_steps(k, false);   // steps jj = kTieSmem / 2 .. 1, chunk by chunk
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_tiefix(const sc_scene &scene, const sc_survivor *surv, const sc_camera &cam, const uint32_t *keys,
                          uint2 *pv, const double *depth64, const unsigned long long *n_dev, int64_t n_max,
                          uint32_t *run_list, double *scratch, Counters *ctr, sc_frame_stats *stats, cudaStream_t st)
{
    if (n_max <= 0) return cudaSuccess;
    const int nsm = sm_count();
    const int64_t blocks = std::min<int64_t>((n_max + 255) / 256, (int64_t)nsm * 16);
    const int64_t hblocks = std::min<int64_t>((n_max + 2047) / 2048, (int64_t)nsm * 8);
    SC_LAUNCH(k_tie_heads, (int)std::max<int64_t>(1, hblocks), 256, 0, st, keys, n_dev, n_max, run_list, ctr);
    // long runs go to the second half of the run-list buffer (runs <= n / 2 <= its half)
    uint32_t *long_list = run_list + (n_max + 1) / 2;
    SC_LAUNCH(k_tie_runs, (int)std::max<int64_t>(1, blocks / 8), 256, 0, st, scene, surv, cam, keys, pv, depth64, n_dev,
              n_max, run_list, long_list, ctr, stats);
    SC_LAUNCH(k_tie_long, nsm * 2, 256, 0, st, scene, surv, cam, keys, pv, depth64, n_dev, n_max, long_list, ctr, stats,
              scratch);
    return cudaGetLastError();
}

}  // namespace sc
