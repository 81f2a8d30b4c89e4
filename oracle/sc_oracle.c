/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference splatcull CPU path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * as the checker.  It is never linked into, called by, or shipped with the
 * product (paper_2511_19202_b200/), which fails loudly without its CUDA
 * library.
 *
 * Numerics contract: float64, compiled with -ffp-contract=off (no FMA), exp /
 * sqrt / ceil / floor from glibc — numba lowers np.exp to glibc's exp for the
 * reference kernels (checked in tests/test_oracle_golden.py), so the raster
 * half is bit-exact with the reference.  Parity pinned against golden vectors
 * produced by the reference itself (oracle/gen_golden.py -> tests/golden/).
 *
 * Raster half (reference: /root/reference/pkg/src/splatcull/):
 *   orc_project      <- _kernels.py:13-134  project_kernel
 *   orc_bin_count /
 *   orc_bin_fill     <- _kernels.py:137-165 bin_tiles
 *   orc_composite    <- _kernels.py:168-275 composite_tiles
 * Scene half (the reference ships no code for it; restated from
 * SPEC.md:325-389 (scene) and SPEC.md:240-323 (nn), pinned decisions in
 * oracle/scene_ref.py and SURVEY.md Appendix B):
 *   orc_scene_cull   frustum test + d_near gate + visibility MLP, per
 *                    (instance, gaussian) pair, survivors in flat order
 *   orc_instantiate  mean' = s R m + t, q' = q_i (x) q, log_s' = log_s + ln s
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Stage (c): projection.  Follows _kernels.py:35-133 operation by operation. */
/* ------------------------------------------------------------------------ */
EXPORT int64_t orc_project(int64_t n, const double *means, const double *log_scales,
                           const double *quats, const double *cam_rot, const double *cam_pos,
                           double focal, double tan_x, double tan_y, double near_,
                           int64_t width, int64_t height, double dilation, double det_eps,
                           double *mean2d, double *cov2d, double *conic, double *depth,
                           double *radius, uint8_t *valid)
{
    const double lim_x = 1.3 * tan_x;
    const double lim_y = 1.3 * tan_y;
    int64_t n_skipped = 0;
#pragma omp parallel for schedule(static) reduction(+ : n_skipped)
    for (int64_t i = 0; i < n; i++) {
        const double *m = means + 3 * i;
        const double *R = cam_rot;
        double tx = R[0] * (m[0] - cam_pos[0]) + R[1] * (m[1] - cam_pos[1]) + R[2] * (m[2] - cam_pos[2]);
        double ty = R[3] * (m[0] - cam_pos[0]) + R[4] * (m[1] - cam_pos[1]) + R[5] * (m[2] - cam_pos[2]);
        double tz = R[6] * (m[0] - cam_pos[0]) + R[7] * (m[1] - cam_pos[1]) + R[8] * (m[2] - cam_pos[2]);
        depth[i] = tz;
        valid[i] = 0;
        if (tz <= near_) {
            mean2d[2 * i] = 0.0; mean2d[2 * i + 1] = 0.0;
            cov2d[3 * i] = dilation; cov2d[3 * i + 1] = 0.0; cov2d[3 * i + 2] = dilation;
            conic[3 * i] = 0.0; conic[3 * i + 1] = 0.0; conic[3 * i + 2] = 0.0;
            radius[i] = 0.0;
            continue;
        }
        double txz = tx / tz;
        double tyz = ty / tz;
        double ctxz = fmin(fmax(txz, -lim_x), lim_x);
        double ctyz = fmin(fmax(tyz, -lim_y), lim_y);
        double fz = focal / tz;
        double m00 = fz * R[0] - fz * ctxz * R[6];
        double m01 = fz * R[1] - fz * ctxz * R[7];
        double m02 = fz * R[2] - fz * ctxz * R[8];
        double m10 = fz * R[3] - fz * ctyz * R[6];
        double m11 = fz * R[4] - fz * ctyz * R[7];
        double m12 = fz * R[5] - fz * ctyz * R[8];

        const double *q = quats + 4 * i;
        double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        double w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
        double r00 = 1.0 - 2.0 * (y * y + z * z);
        double r01 = 2.0 * (x * y - w * z);
        double r02 = 2.0 * (x * z + w * y);
        double r10 = 2.0 * (x * y + w * z);
        double r11 = 1.0 - 2.0 * (x * x + z * z);
        double r12 = 2.0 * (y * z - w * x);
        double r20 = 2.0 * (x * z - w * y);
        double r21 = 2.0 * (y * z + w * x);
        double r22 = 1.0 - 2.0 * (x * x + y * y);

        const double *ls = log_scales + 3 * i;
        double s0 = exp(2.0 * ls[0]);
        double s1 = exp(2.0 * ls[1]);
        double s2 = exp(2.0 * ls[2]);

        double g00 = r00 * r00 * s0 + r01 * r01 * s1 + r02 * r02 * s2;
        double g01 = r00 * r10 * s0 + r01 * r11 * s1 + r02 * r12 * s2;
        double g02 = r00 * r20 * s0 + r01 * r21 * s1 + r02 * r22 * s2;
        double g11 = r10 * r10 * s0 + r11 * r11 * s1 + r12 * r12 * s2;
        double g12 = r10 * r20 * s0 + r11 * r21 * s1 + r12 * r22 * s2;
        double g22 = r20 * r20 * s0 + r21 * r21 * s1 + r22 * r22 * s2;

        double u0 = m00 * g00 + m01 * g01 + m02 * g02;
        double u1 = m00 * g01 + m01 * g11 + m02 * g12;
        double u2 = m00 * g02 + m01 * g12 + m02 * g22;
        double v0 = m10 * g00 + m11 * g01 + m12 * g02;
        double v1 = m10 * g01 + m11 * g11 + m12 * g12;
        double v2 = m10 * g02 + m11 * g12 + m12 * g22;
        double a = u0 * m00 + u1 * m01 + u2 * m02 + dilation;
        double b = u0 * m10 + u1 * m11 + u2 * m12;
        double c = v0 * m10 + v1 * m11 + v2 * m12 + dilation;

        mean2d[2 * i] = focal * txz + (double)(width - 1) / 2.0;
        mean2d[2 * i + 1] = focal * tyz + (double)(height - 1) / 2.0;
        cov2d[3 * i] = a; cov2d[3 * i + 1] = b; cov2d[3 * i + 2] = c;

        double det = a * c - b * b;
        if (det <= det_eps) {
            conic[3 * i] = 0.0; conic[3 * i + 1] = 0.0; conic[3 * i + 2] = 0.0;
            radius[i] = 0.0;
            n_skipped += 1;
            continue;
        }
        conic[3 * i] = c / det;
        conic[3 * i + 1] = -b / det;
        conic[3 * i + 2] = a / det;
        double mid = 0.5 * (a + c);
        double disc = mid * mid - det;
        double lam = mid + sqrt(disc > 0.0 ? disc : 0.0);
        double r3 = ceil(3.0 * sqrt(lam));
        radius[i] = r3;
        if (r3 > 0.0) valid[i] = 1;
    }
    return n_skipped;
}

/* ------------------------------------------------------------------------ */
/* Stage (d): counting sort into tile segments (_kernels.py:137-165).       */
/* counts has n_tiles + 1 slots; orc_bin_count fills the inclusive prefix.  */
/* ------------------------------------------------------------------------ */
EXPORT void orc_bin_count(int64_t m, const int64_t *order_idx, const int64_t *tx0, const int64_t *tx1,
                          const int64_t *ty0, const int64_t *ty1, int64_t n_tiles_x, int64_t n_tiles,
                          int64_t *counts)
{
    memset(counts, 0, sizeof(int64_t) * (size_t)(n_tiles + 1));
    for (int64_t k = 0; k < m; k++) {
        int64_t i = order_idx[k];
        for (int64_t tyy = ty0[i]; tyy < ty1[i]; tyy++) {
            int64_t base = tyy * n_tiles_x;
            for (int64_t txx = tx0[i]; txx < tx1[i]; txx++) counts[base + txx + 1] += 1;
        }
    }
    for (int64_t t = 0; t < n_tiles; t++) counts[t + 1] += counts[t];
}

EXPORT void orc_bin_fill(int64_t m, const int64_t *order_idx, const int64_t *tx0, const int64_t *tx1,
                         const int64_t *ty0, const int64_t *ty1, int64_t n_tiles_x, int64_t n_tiles,
                         const int64_t *counts, int64_t *entry_idx)
{
    int64_t *cursors = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_tiles > 0 ? n_tiles : 1));
    memcpy(cursors, counts, sizeof(int64_t) * (size_t)n_tiles);
    for (int64_t k = 0; k < m; k++) {
        int64_t i = order_idx[k];
        for (int64_t tyy = ty0[i]; tyy < ty1[i]; tyy++) {
            int64_t base = tyy * n_tiles_x;
            for (int64_t txx = tx0[i]; txx < tx1[i]; txx++) {
                int64_t t = base + txx;
                entry_idx[cursors[t]] = i;
                cursors[t] += 1;
            }
        }
    }
    free(cursors);
}

/* ------------------------------------------------------------------------ */
/* Stage (e): per-tile front-to-back compositing (_kernels.py:190-275).     */
/* ------------------------------------------------------------------------ */
EXPORT void orc_composite(int64_t n_active, const int64_t *active_tiles, const int64_t *tile_start,
                          const int64_t *tile_end, const int64_t *entry_idx, const double *mean2d,
                          const double *conic, const double *opacity, const double *log_opacity,
                          const double *color, const double *radius, int64_t height, int64_t width,
                          int64_t tile_size, int64_t n_tiles_x, double stop_t, double min_alpha,
                          double log_min_alpha, int32_t record, double *image, double *trans,
                          double *contrib_sum, double *entry_contrib)
{
#pragma omp parallel
    {
        int64_t cap = tile_size * tile_size;
        double *t_loc = (double *)malloc(sizeof(double) * (size_t)cap);
        int64_t *live_x = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
        int64_t *live_y = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
#pragma omp for schedule(dynamic, 4)
        for (int64_t ti = 0; ti < n_active; ti++) {
            int64_t tile = active_tiles[ti];
            int64_t ty = tile / n_tiles_x;
            int64_t tx = tile - ty * n_tiles_x;
            int64_t y0 = ty * tile_size, x0 = tx * tile_size;
            int64_t th = tile_size < height - y0 ? tile_size : height - y0;
            int64_t tw = tile_size < width - x0 ? tile_size : width - x0;
            int64_t k = 0;
            for (int64_t ly = 0; ly < th; ly++)
                for (int64_t lx = 0; lx < tw; lx++) {
                    t_loc[ly * tw + lx] = 1.0;
                    live_y[k] = ly; live_x[k] = lx; k++;
                }
            int64_t n_live = th * tw;
            for (int64_t e = tile_start[ti]; e < tile_end[ti]; e++) {
                if (n_live == 0) break;
                int64_t g = entry_idx[e];
                double op = opacity[g];
                if (op < min_alpha) continue;
                double p_min = log_min_alpha - log_opacity[g];
                double mx = mean2d[2 * g], my = mean2d[2 * g + 1];
                double r = radius[g];
                int64_t lya = (int64_t)floor(my - r) - y0; if (lya < 0) lya = 0;
                int64_t lyb = (int64_t)floor(my + r) + 1 - y0; if (lyb > th - 1) lyb = th - 1;
                int64_t lxa = (int64_t)floor(mx - r) - x0; if (lxa < 0) lxa = 0;
                int64_t lxb = (int64_t)floor(mx + r) + 1 - x0; if (lxb > tw - 1) lxb = tw - 1;
                double half_a = 0.5 * conic[3 * g];
                double b = conic[3 * g + 1];
                double half_c = 0.5 * conic[3 * g + 2];
                double cr = color[3 * g], cg = color[3 * g + 1], cb = color[3 * g + 2];
                double cmax = 0.0;
                int64_t j = 0;
                while (j < n_live) {
                    int64_t ly = live_y[j], lx = live_x[j];
                    if (ly < lya || ly > lyb || lx < lxa || lx > lxb) { j++; continue; }
                    double dx = (double)(x0 + lx) - mx;
                    double dy = (double)(y0 + ly) - my;
                    double power = -(half_a * dx * dx + half_c * dy * dy) - b * dx * dy;
                    if (power > 0.0 || power < p_min) { j++; continue; }
                    double alpha = op * exp(power);
                    if (alpha > 0.99) alpha = 0.99;
                    double t_cur = t_loc[ly * tw + lx];
                    double contrib = alpha * t_cur;
                    int64_t py = y0 + ly, px = x0 + lx;
                    double *pix = image + 3 * (py * width + px);
                    pix[0] += contrib * cr;
                    pix[1] += contrib * cg;
                    pix[2] += contrib * cb;
                    if (record) {
                        contrib_sum[py * width + px] += contrib;
                        if (contrib > cmax) cmax = contrib;
                    }
                    double t_new = t_cur * (1.0 - alpha);
                    t_loc[ly * tw + lx] = t_new;
                    if (t_new < stop_t) {
                        n_live -= 1;
                        live_y[j] = live_y[n_live];
                        live_x[j] = live_x[n_live];
                    } else {
                        j++;
                    }
                }
                if (record) entry_contrib[e] = cmax;
            }
            for (int64_t ly = 0; ly < th; ly++)
                for (int64_t lx = 0; lx < tw; lx++) trans[(y0 + ly) * width + x0 + lx] = t_loc[ly * tw + lx];
        }
        free(t_loc); free(live_x); free(live_y);
    }
}

/* ------------------------------------------------------------------------ */
/* Scene half.  Decisions pinned in oracle/scene_ref.py.    */
/* ------------------------------------------------------------------------ */

/* Instance record shared with oracle/scene_ref.py (all f64, host-derived). */
typedef struct {
    double R[9];      /* rotation matrix of the instance quaternion (row-major) */
    double t[3];      /* translation */
    double q[4];      /* normalised instance quaternion (w, x, y, z) */
    double s;         /* uniform scale */
    double ln_s;      /* log(s), host libm */
    double corr;      /* (f_train / cam.focal) / s  (Eq. 2 factor, per frame) */
    double fwd_local[3]; /* R^T cam.forward (per frame) */
    int64_t asset;    /* asset index */
} orc_instance;

typedef struct {
    int64_t offset, count;   /* into the concatenated gaussian arrays */
    double d_near, d_far, bound_radius;
    int64_t model;           /* -1: no visibility model */
} orc_asset;

typedef struct {
    double pos[3], rot[9];
    double focal, tan_x, tan_y, near_;
    int64_t width, height, tile_size;
} orc_camera;

/* B2: instanced mean, f64 scalar order, rounded to f32 (Asset dtype). */
static inline void inst_mean(const orc_instance *in, const float *m, float *out)
{
    for (int k = 0; k < 3; k++) {
        double v = in->R[3 * k] * (double)m[0] + in->R[3 * k + 1] * (double)m[1] + in->R[3 * k + 2] * (double)m[2];
        out[k] = (float)(in->s * v + in->t[k]);
    }
}

static inline void inst_quat(const orc_instance *in, const float *q, float *out)
{
    double w1 = in->q[0], x1 = in->q[1], y1 = in->q[2], z1 = in->q[3];
    double w2 = q[0], x2 = q[1], y2 = q[2], z2 = q[3];
    out[0] = (float)(w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2);
    out[1] = (float)(w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2);
    out[2] = (float)(w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2);
    out[3] = (float)(w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2);
}

EXPORT void orc_instantiate(int64_t n_surv, const int64_t *surv_inst, const int64_t *surv_gid,
                            const orc_instance *inst, const float *means, const float *log_scales,
                            const float *quats, const float *opacity_logits, const float *sh,
                            int64_t sh_stride, float *o_means, float *o_log_scales, float *o_quats,
                            float *o_opacity, float *o_sh)
{
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n_surv; k++) {
        const orc_instance *in = inst + surv_inst[k];
        int64_t g = surv_gid[k];
        inst_mean(in, means + 3 * g, o_means + 3 * k);
        for (int c = 0; c < 3; c++) o_log_scales[3 * k + c] = (float)((double)log_scales[3 * g + c] + in->ln_s);
        inst_quat(in, quats + 4 * g, o_quats + 4 * k);
        o_opacity[k] = opacity_logits[g];
        memcpy(o_sh + sh_stride * k, sh + sh_stride * g, sizeof(float) * (size_t)sh_stride);
    }
}

/* B3 margin pad in pixels: radius = ceil(3 sqrt(lambda)) <= 3 sigma (f / tz) G + 3 sqrt(dilation) + 1,
 * so max(3, 3 sqrt(dilation) + 1 + 1e-6) covers every splat the rasterizer can pass (3 px at the
 * default dilation 0.3).  Same expression as the device (common.cuh margin_pad). */
EXPORT double orc_margin_pad(double dilation)
{
    double p = 3.0 * sqrt(dilation > 0.0 ? dilation : 0.0) + 1.0 + 1e-6;
    return p > 3.0 ? p : 3.0;
}

/* B3 frustum predicate on the f32-rounded instanced mean (see scene_ref.py). */
static inline int frustum_pass(const orc_camera *cam, const double mw[3], double sigma_w, double G, double pad,
                               int strict, double *out_t /* tx, ty, tz */)
{
    const double *R = cam->rot;
    const double *c = cam->pos;
    double tx = R[0] * (mw[0] - c[0]) + R[1] * (mw[1] - c[1]) + R[2] * (mw[2] - c[2]);
    double ty = R[3] * (mw[0] - c[0]) + R[4] * (mw[1] - c[1]) + R[5] * (mw[2] - c[2]);
    double tz = R[6] * (mw[0] - c[0]) + R[7] * (mw[1] - c[1]) + R[8] * (mw[2] - c[2]);
    out_t[0] = tx; out_t[1] = ty; out_t[2] = tz;
    if (tz <= cam->near_) return 0;
    double mx = cam->focal * (tx / tz) + (double)(cam->width - 1) / 2.0;
    double my = cam->focal * (ty / tz) + (double)(cam->height - 1) / 2.0;
    if (strict) {
        return mx >= 0.0 && mx <= (double)(cam->width - 1) && my >= 0.0 && my <= (double)(cam->height - 1);
    }
    double rb = 3.0 * (cam->focal / tz) * sigma_w * G + pad;
    double tw = (double)(cam->tile_size * ((cam->width + cam->tile_size - 1) / cam->tile_size));
    double th = (double)(cam->tile_size * ((cam->height + cam->tile_size - 1) / cam->tile_size));
    return (mx + rb >= 0.0) && (mx - rb < tw) && (my + rb >= 0.0) && (my - rb < th);
}

/* Dense ReLU MLP in f64: widths w[0..n_layers], weights row-major [out][in]. */
static void mlp_forward(const double *params, const int64_t *widths, int64_t n_layers, const double *x,
                        double *out)
{
    double buf0[64], buf1[64];
    const double *in = x;
    double *cur = buf0;
    const double *p = params;
    for (int64_t l = 0; l < n_layers; l++) {
        int64_t ni = widths[l], no = widths[l + 1];
        const double *W = p;
        const double *b = p + ni * no;
        double *dst = (l == n_layers - 1) ? out : cur;
        for (int64_t o = 0; o < no; o++) {
            double acc = 0.0;
            for (int64_t i = 0; i < ni; i++) acc += W[o * ni + i] * in[i];
            acc += b[o];
            if (l < n_layers - 1 && acc < 0.0) acc = 0.0;
            dst[o] = acc;
        }
        p += ni * no + no;
        in = dst;
        cur = (cur == buf0) ? buf1 : buf0;
    }
}

/*
 * Per (instance, gaussian) pair: frustum test, d_near gate, visibility MLP.
 * Writes keep[pair] (1 = survivor), and for queried pairs logit[pair]
 * (NaN when not queried).  Pair index = inst_pair_offset[i] + gid - asset.offset.
 * flags[pair]: bit0 frustum pass, bit1 queried.
 */
EXPORT void orc_scene_cull(int64_t n_inst, const orc_instance *inst, const int64_t *inst_pair_offset,
                           const orc_asset *assets, const orc_camera *cam, const float *means,
                           const float *sigma_max, const double *features, const double *model_params,
                           const int64_t *model_param_offset, const int64_t *vis_widths, int64_t vis_layers,
                           double G, double dilation, int32_t strict, int32_t use_models,
                           double logit_threshold, uint8_t *keep, uint8_t *flags, double *logit)
{
    const double pad = orc_margin_pad(dilation);
    for (int64_t i = 0; i < n_inst; i++) {
        const orc_instance *in = inst + i;
        const orc_asset *a = assets + in->asset;
        const double *params = (use_models && a->model >= 0) ? model_params + model_param_offset[a->model] : NULL;
        int64_t base = inst_pair_offset[i];
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < a->count; j++) {
            int64_t g = a->offset + j;
            int64_t pair = base + j;
            float mf[3];
            inst_mean(in, means + 3 * g, mf);
            double mw[3] = {(double)mf[0], (double)mf[1], (double)mf[2]};
            double tcam[3];
            double sigma_w = in->s * (double)sigma_max[g];
            keep[pair] = 0;
            flags[pair] = 0;
            logit[pair] = NAN;
            if (!frustum_pass(cam, mw, sigma_w, G, pad, strict, tcam)) continue;
            flags[pair] = 1;
            if (params == NULL) { keep[pair] = 1; continue; }
            double dx = mw[0] - cam->pos[0], dy = mw[1] - cam->pos[1], dz = mw[2] - cam->pos[2];
            double d_r = sqrt(dx * dx + dy * dy + dz * dz);
            double d_t = d_r * in->corr;
            if (!(d_t >= a->d_near)) { keep[pair] = 1; continue; }
            flags[pair] |= 2;
            double x[16];
            const double *m = NULL;
            (void)m;
            for (int k = 0; k < 3; k++) x[k] = (double)means[3 * g + k] / a->bound_radius;
            double inv = 1.0 / d_r;
            for (int k = 0; k < 3; k++)
                x[3 + k] = (in->R[k] * dx + in->R[3 + k] * dy + in->R[6 + k] * dz) * inv;
            double dn = 2.0 * (d_t - a->d_near) / (a->d_far - a->d_near) - 1.0;
            x[6] = dn < -1.0 ? -1.0 : (dn > 1.0 ? 1.0 : dn);
            for (int k = 0; k < 3; k++) x[7 + k] = in->fwd_local[k];
            for (int k = 0; k < 6; k++) x[10 + k] = features[6 * g + k];
            double lg;
            mlp_forward(params, vis_widths, vis_layers, x, &lg);
            logit[pair] = lg;
            keep[pair] = lg >= logit_threshold;
        }
    }
}

/* Batched MLP forward (config-4 sweep and encode_features reference). */
EXPORT void orc_mlp_forward(int64_t n, const double *params, const int64_t *widths, int64_t n_layers,
                            const double *x, double *out)
{
    int64_t ni = widths[0], no = widths[n_layers];
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; r++) mlp_forward(params, widths, n_layers, x + r * ni, out + r * no);
}
