/*
 * splatcull_b200 — C ABI of the B200 (sm_100a) instanced 3DGS render path
 * with neural occlusion culling.
 *
 * The reference (arxiv 2511.19202 desk-scale package `splatcull`) is pure
 * Python + numba; it has no C ABI.  Each entry point below replaces one
 * function of the reference's Python/numba path; the Python host package
 * (paper_2511_19202_b200) binds them with ctypes and keeps the reference's
 * Python names.  Replaced reference interfaces:
 *
 *   sc_render_composed  <- scene.render_composed
 *                          (+ raster.render, sc/raster.py:240-339, as the
 *                           single-identity-instance / no-cull special case)
 *   sc_cull_mlp         <- render_composed steps (1)-(2): frustum test +
 *                          d_near gate + visibility MLP
 *   sc_project          <- project_kernel                   sc/_kernels.py:13-134
 *                          + eval_sh_colors / sigmoid       sc/raster.py:198-226, sc/asset.py:44-51
 *                          + radius clip / tile rects       sc/raster.py:287-316
 *   sc_bin_sort         <- argsort(depth, stable)           sc/raster.py:319
 *                          + bin_tiles                      sc/_kernels.py:137-165
 *   sc_blend            <- composite_tiles + finish()       sc/_kernels.py:168-275, sc/raster.py:267-282
 *   sc_vis_mlp_forward  <- nn.forward (16->32->32->1)
 *   sc_encode_features  <- nn.encode_features (14->32->32->6) SPEC.md:286-294
 *   sc_visibility_labels_or <- sampling.visible_labels      sc/sampling.py:206-213
 *
 * Conventions
 *   - every pointer in the sc_* structs is DEVICE memory unless noted;
 *     the library never allocates device memory: the caller passes all
 *     buffers (workspace sized by sc_workspace_bytes), so the caller's
 *     allocator accounts for peak VRAM;
 *   - all calls are asynchronous and stream-ordered on `stream`
 *     (a cudaStream_t passed as void*; NULL = legacy default stream);
 *   - return value: SC_OK or an SC_ERR_* code, message in sc_last_error()
 *     (thread-local).  Data-dependent overflow (survivors or tile entries
 *     beyond the workspace capacity) is reported in sc_frame_stats.overflow
 *     after the stream completes; the caller grows the workspace and
 *     re-renders (reference kernels report conditioning drops as counts the
 *     same way, sc/_kernels.py:117-124);
 *   - thread-compatible: one workspace per concurrent stream.
 */
#ifndef SPLATCULL_B200_H
#define SPLATCULL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_ABI_VERSION 3

#if defined(__GNUC__)
#define SC_API __attribute__((visibility("default")))
#else
#define SC_API
#endif

enum {
    SC_OK = 0,
    SC_ERR_INVALID = 1,   /* bad argument (shape, size, option) */
    SC_ERR_CUDA = 2,      /* CUDA launch / runtime error */
    SC_ERR_UNSUPPORTED = 3
};

/* frustum_mode */
enum {
    SC_FRUSTUM_MARGIN = 0,  /* conservative: superset of splats the rasterizer passes (default) */
    SC_FRUSTUM_STRICT = 1,  /* paper mode: mean must project inside the image */
    SC_FRUSTUM_OFF = 2      /* no culling (plain raster.render) */
};

/* Pinhole camera (reference raster.Camera, sc/raster.py:40-99).  Host struct. */
typedef struct sc_camera {
    double pos[3];
    double rot[9];      /* world->camera, rows right, down, forward */
    double focal;       /* height / (2 tan(fov_y / 2)) */
    double tan_x, tan_y;
    double near_;
    int32_t width, height;
} sc_camera;

/* Render options (reference render() keywords, sc/raster.py:240-251). Host struct. */
typedef struct sc_opts {
    int32_t tile_size;            /* reference tile edge in pixels, 1..65535 (default 16; the image
                                     depends on it, sc/raster.py:297-311, sc/_kernels.py:224-227);
                                     screen bands need 16 */
    int32_t sh_degree_eval;       /* -1: use each asset's degree */
    int32_t record_contributions; /* per-splat max contribution + per-pixel sum */
    int32_t use_mlp;              /* 0: no MLP gate ("Ours w/o MLP") */
    int32_t frustum_mode;         /* SC_FRUSTUM_* */
    int32_t exact_projection;     /* 1: all-f64 projection; 0: f32 covariance with exact f64
                                     fallback whenever the radius / clip decision is ambiguous */
    double radius_clip;           /* <= 0: off */
    double stop_transmittance;    /* 1/255 */
    double background[3];         /* (1, 1, 1) */
    double dilation;              /* 0.3 */
    double frustum_G;             /* Jacobian bound factor */
    /* screen band [band_y0, band_y1) in pixel rows, band_y0 a multiple of 16
     * (band_y1 may be the image height); band_y1 <= 0: the whole image.  Only
     * the band's pixels are written; they are identical to the whole-image
     * render (the band's sub-frustum is a conservative superset). */
    int32_t band_y0, band_y1;
} sc_opts;

/*
 * Scene, uploaded once.  Gaussians of all assets are concatenated; asset a
 * owns [assets[a].offset, assets[a].offset + assets[a].count).
 */
typedef struct sc_asset_rec {
    int64_t offset, count;
    double d_near, d_far;        /* MLP gate + min-max normalisation (model norm) */
    double inv_mean_scale;       /* 1 / model.mean_scale */
    double f_train;              /* training focal (Eq. 2) */
    double bound_local;          /* max |mean| over the asset (local units) */
    double sigma_max;            /* max exp(max log_scale) over the asset */
    int32_t model;               /* index into sc_scene.vis_weights, -1 = none */
    int32_t sh_degree;
    float logit_threshold;       /* keep iff logit >= this */
    int32_t reserved0;
} sc_asset_rec;

/* Per instance, flat order (asset-major, then instance order). */
typedef struct sc_instance_rec {
    double R[9];                 /* rotation of the normalised instance quaternion */
    double t[3];
    double q[4];                 /* normalised (w, x, y, z) */
    double s, ln_s;              /* uniform scale, log(s) (host libm) */
    int32_t asset;
    int32_t reserved0;
} sc_instance_rec;

/* Visibility-MLP weights of one model, device layout (fp16 = uint16 bits). */
#define SC_VIS_HIDDEN 32
typedef struct sc_vis_weights {
    uint16_t w1[SC_VIS_HIDDEN * 16];            /* [out][in] fp16 */
    uint16_t w2[SC_VIS_HIDDEN * SC_VIS_HIDDEN]; /* [out][in] fp16 */
    float b1[SC_VIS_HIDDEN];
    float b2[SC_VIS_HIDDEN];
    float w3[SC_VIS_HIDDEN];
    float b3;
    float reserved[31];
} sc_vis_weights;

typedef struct sc_scene {
    /* gaussians, n_gauss each */
    const float *mean_opa;       /* float4 (x, y, z, opacity_logit) */
    const float *quat;           /* float4 (w, x, y, z) */
    const float *scale_smax;     /* float4 (log_s0, log_s1, log_s2, sigma_max) */
    const float *sh;             /* [n_gauss][sh_stride] f32, coefficient-major then RGB */
    const uint16_t *features;    /* [n_gauss][8] fp16 (6 used) */
    int64_t n_gauss;
    int32_t sh_stride;           /* floats per gaussian = 3 (deg+1)^2 of the max degree */
    int32_t n_assets;
    const sc_asset_rec *assets;  /* [n_assets] */
    const sc_instance_rec *instances; /* [n_instances] */
    int64_t n_instances;
    const sc_vis_weights *vis_weights; /* [n_models] */
    int32_t n_models;
    int32_t reserved0;
    int64_t n_pairs;             /* sum over instances of their asset's count (workspace check) */
    /* [n_gauss] float4 per gaussian, view-independent appearance computed once
     * in f64 like the reference and rounded: x = p_min = ln(1/255) - ln(sigmoid(
     * opacity_logit)), +inf when opacity < 1/255 (sc/_kernels.py:215-219);
     * y, z = the degree-0 colour clip(C0 f_dc + 0.5, 0, 1) as fp16 bits (r | g << 16,
     * b); w = 0 */
    const float *appear;
} sc_scene;

/* Device-side counters of one frame (copy back with the stream). */
typedef struct sc_frame_stats {
    int64_t instances_visible;   /* after the per-instance bounding-sphere cull */
    int64_t pairs_tested;        /* (gaussian, instance) pairs reaching the per-gaussian test */
    int64_t frustum_passed;
    int64_t mlp_queried;
    int64_t mlp_culled;
    int64_t survivors;           /* instantiated = frustum_passed - mlp_culled */
    int64_t passed;              /* valid, not radius-clipped, on a tile (reference passed_count) */
    int64_t skipped;             /* det <= 1e-12 conditioning drops */
    int64_t entries;             /* tile entries E */
    int64_t used;                /* splats with contribution_max > 0 (record mode) */
    int64_t max_tie_run;         /* longest run of equal f32 depth keys (tie-fix work) */
    int64_t overflow;            /* bit0 survivors, bit1 entries, bit2 block lists, bit3 scene pairs beyond
                                    the workspace's max_pairs: re-render with more capacity */
    int64_t block_entries;       /* frame path: (splat, 8x4 pixel block) entries binned for the blend */
    int64_t exact_fallbacks;     /* projections that fell back to the all-f64 path (exact_projection = 0) */
    int64_t reserved[2];
} sc_frame_stats;

/* Survivor = (instance index, gaussian index within its asset). */
typedef struct sc_survivor { uint32_t inst, gid; } sc_survivor;

/* Per-survivor splat record consumed by the blend (32 B = one sector).
 * opacity is implied: alpha = min(0.99, exp(power - p_min) / 255), which equals
 * opacity * exp(power) for p_min = log(1/255) - log(opacity). */
typedef struct sc_splat {
    float mx, my;                /* pixel-space mean */
    float half_a, b, half_c;     /* 0.5 conic_a, conic_b, 0.5 conic_c */
    float p_min;                 /* log(1/255) - log(opacity); +inf = skipped (opacity < 1/255) */
    uint16_t rgb[3];             /* fp16 colour */
    uint16_t reserved;
} sc_splat;

/* Per-survivor pixel window [x0, x1] x [y0, y1] (inclusive, absolute pixels):
 * the reference window (sc/_kernels.py:224-227) intersected with the
 * alpha >= 1/255 support box and the tile rectangle, computed in f64. */
typedef struct sc_window { int16_t x0, x1, y0, y1; } sc_window;

/* Bytes of workspace for the given capacities (align 256).  Host call. */
SC_API size_t sc_workspace_bytes(int64_t n_instances, int64_t max_pairs, int64_t cap_survivors,
                          int64_t cap_entries, int32_t width, int32_t height, int32_t tile_size);

/* Optional frame-path internals copied out for parity tests (all device, NULL
 * to skip each): the depth order and the per-(16x16 tile, 8x4 block) lists
 * the blend walks.  Block b of tile t has id 8 t + b, b = 2 row + col (x in
 * [8 col, 8 col + 7], y in [4 row, 4 row + 3] inside the 16x16 tile). */
typedef struct sc_frame_debug {
    uint32_t *order;          /* [cap_survivors]: passed survivors in (depth, index) order (stats.passed) */
    uint32_t *block_offsets;  /* [8 n_tiles16 + 1]: list of block id k = [offsets[k], offsets[k + 1]) */
    uint32_t *block_entries;  /* [cap_entries]: survivor index per block entry (stats.block_entries) */
    uint32_t *block_codes;    /* [cap_entries]: block id << 10 | block-relative window
                                 x0 | x1 << 3 | y0 << 6 | y1 << 8 */
} sc_frame_debug;

typedef struct sc_frame_out {
    float *image;                /* [H][W][3] f32, background composited */
    float *trans;                /* [H][W] f32 final transmittance */
    float *contrib_sum;          /* [H][W] f32 or NULL (record mode) */
    float *contrib_max;          /* [cap_survivors] f32 or NULL (record mode) */
    sc_frame_stats *stats;       /* device */
    sc_survivor *survivors;      /* optional device copy-out [cap_survivors] or NULL */
    /* optional stage timing: cudaEvent_t handles (host array), recorded on the
     * stream at [0] frame start, [1] after cull+MLP, [2] after projection,
     * [3] after sort/binning, [4] after blend.  NULL to skip. */
    void *const *stage_events;
    int32_t n_stage_events;
    int32_t reserved0;
    const sc_frame_debug *debug; /* optional (NULL) */
} sc_frame_out;

#define SC_STAGE_EVENTS 5

typedef struct sc_workspace {
    void *base;                  /* device, sc_workspace_bytes() bytes */
    size_t bytes;
    int64_t n_instances, max_pairs;   /* as passed to sc_workspace_bytes */
    int64_t cap_survivors, cap_entries;
} sc_workspace;

/* Whole frame: cull + MLP -> project -> sort/bin -> blend. */
SC_API int sc_render_composed(const sc_scene *scene, const sc_camera *cam, const sc_opts *opts,
                       const sc_workspace *ws, const sc_frame_out *out, void *stream);

/* Stages (c)-(e) of the frame path on an explicit survivor list (device,
 * n <= ws->cap_survivors, e.g. the oracle's cull): the same kernels as
 * sc_render_composed after its cull, so stage-level parity tests can inject
 * survivors into the benchmarked path. */
SC_API int sc_render_survivors(const sc_scene *scene, const sc_survivor *survivors, int64_t n, const sc_camera *cam,
                        const sc_opts *opts, const sc_workspace *ws, const sc_frame_out *out, void *stream);

/* Stage (a)+(b): survivors in flat (instance, gaussian) order + stats. */
SC_API int sc_cull_mlp(const sc_scene *scene, const sc_camera *cam, const sc_opts *opts,
                const sc_workspace *ws, sc_survivor *survivors, int64_t cap_survivors,
                sc_frame_stats *stats, void *stream);

/*
 * Stage (c) on an explicit survivor list (host count n).  Optional f64 debug
 * outputs (NULL to skip) let tests compare with the oracle bit for bit:
 * dbg_f64 = [n][8] (mx, my, conic a, b, c, depth, radius, cov det);
 * dbg_rect = [n][4] int32 (tx0, tx1, ty0, ty1), dbg_flags = [n] u8
 * (bit0 valid after clip, bit1 passed).
 */
SC_API int sc_project(const sc_scene *scene, const sc_survivor *survivors, int64_t n,
               const sc_camera *cam, const sc_opts *opts, sc_splat *splats, sc_window *windows,
               double *dbg_f64, int32_t *dbg_rect, uint8_t *dbg_flags, sc_frame_stats *stats, void *stream);

/*
 * Stages (c)+(d) on an explicit survivor list: projection, (depth, index)
 * order, tile binning.  Writes splats [n], order_idx [n] (passed survivors
 * in (depth, index) order, stats.passed of them), entry_idx
 * [ws->cap_entries] (survivor index per entry, tile-major, depth order inside
 * a tile) and tile_offsets [n_tiles + 1] (the reference's `counts`, uint32),
 * stats.entries.
 */
SC_API int sc_bin_sort(const sc_scene *scene, const sc_survivor *survivors, int64_t n,
                const sc_camera *cam, const sc_opts *opts, const sc_workspace *ws,
                sc_splat *splats, sc_window *windows, uint32_t *entry_idx, uint32_t *tile_offsets,
                uint32_t *order_idx, sc_frame_stats *stats, void *stream);

/*
 * Stage (e) on explicit inputs: splats / windows [n_splats] (sc_project
 * output), entry_idx [E] and tile_offsets [n_tiles + 1] (uint32; e.g. the
 * oracle's bin_tiles output) -> image / trans (+ contrib_sum / contrib_max).
 */
SC_API int sc_blend(const sc_splat *splats, const sc_window *windows, int64_t n_splats,
             const uint32_t *entry_idx, const uint32_t *tile_offsets, const sc_camera *cam,
             const sc_opts *opts, const sc_frame_out *out, void *stream);

/* Batched visibility MLP on materialised inputs x [n][16] f32 -> logits [n]. */
SC_API int sc_vis_mlp_forward(const sc_vis_weights *w, const float *x, int64_t n, float *logits,
                       void *stream);

/* Visibility labels of one render (sc/sampling.py:206-213, visible_labels):
 * label_bits[i / 32] |= (contrib_max[i] > 0) << (i % 32) for i < n, i.e. the
 * OR over a view's main and auxiliary renders accumulates in place; the words
 * read as bytes are numpy.packbits(labels, bitorder="little").  contrib_max is
 * sc_frame_out.contrib_max of a record-mode render (survivor order = gaussian
 * order for the single identity instance without culling). */
SC_API int sc_visibility_labels_or(const float *contrib_max, int64_t n, uint32_t *label_bits, void *stream);

/* Feature MLP 14->32->32->6: params f32 (W1,b1,W2,b2,W3,b3 row-major [out][in]),
 * inputs x [n][14] f32 -> features [n][8] fp16 (6 used, 2 zero). */
SC_API int sc_encode_features(const float *params, const float *x, int64_t n, uint16_t *features,
                       void *stream);

SC_API const char *sc_last_error(void);
SC_API int sc_abi_version(void);
/* Number of CUDA kernels this library launched since load (evidence counter). */
SC_API int64_t sc_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SPLATCULL_B200_H */
