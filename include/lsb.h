/*
 * lsb.h — C ABI of the B200 splat hot path (libsplat_b200.so).
 *
 * Drop-in boundary for the reference package livsplat (arXiv 2501.08672
 * desk-scale reimplementation).  The reference has no native boundary of its
 * own: its hot path is the Python entry points render / backward / pose_rows
 * (raster.py:212,309,450), photometric_loss / optimize_window (optimize.py:48,
 * 122), visual_measurement's H/b (estimator.py:260-323) and the HashOctree
 * batch operations (voxmap.py:99-251).  Each function below replaces the
 * numba/numpy body of one of those entry points; the Python host layer
 * (paper_2501_08672_b200/) keeps the reference's names and signatures and
 * binds this header with ctypes.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers allocated by the caller (torch
 *    tensors on the host side).  The library never allocates or frees caller
 *    memory; scratch lives in a caller-provided workspace whose size comes
 *    from lsb_workspace_bytes().
 *  - Every call is asynchronous and stream-ordered on `stream` (a
 *    cudaStream_t passed as void*).  Only the *_counts / *_read functions
 *    synchronise, and they say so.
 *  - Return value: LSB_OK or an error code; lsb_last_error() gives a
 *    thread-local message.  The host layer maps codes to the reference's
 *    exception types (errors.py): LSB_EMISSING_CACHE -> MissingCache,
 *    LSB_EINVAL -> ValueError, LSB_ECAPACITY -> retry with a larger workspace.
 *  - No global mutable state: concurrent calls on different streams with
 *    different workspaces are safe (reference SPEC.md:322).
 */
#ifndef LSB_H
#define LSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSB_ABI_VERSION 1

enum lsb_status {
    LSB_OK = 0,
    LSB_EINVAL = 1,          /* bad argument                                  */
    LSB_ECAPACITY = 2,       /* workspace capacity exceeded: grow and retry   */
    LSB_ECUDA = 3,           /* CUDA runtime error                            */
    LSB_EMISSING_CACHE = 4   /* backward on a render without its state        */
};

/* PinholeCamera (geometry.py:231-244). */
typedef struct lsb_camera {
    double fx, fy, cx, cy;
    int32_t width, height;
} lsb_camera;

/* RasterSettings (raster.py:24-34). */
typedef struct lsb_settings {
    double near_plane;         /* near                                     */
    double dilation;           /* px^2 added to both 2-D eigenvalues       */
    double alpha_clamp;
    double transmittance_min;
    double footprint_sigma;
    double alpha_cut;
    double max_footprint_px;
    double background[3];
    int32_t sh_degree;
    /* Tile-list mode.  0: every splat whose footprint bbox touches the tile
     * (the reference's per-pixel CSR lists, _kernels.py:21-59; n_contrib is
     * the reference's processed-entry count).  1 (only with alpha_cut > 0):
     * only splats whose alpha >= alpha_cut ellipse can reach a pixel of the
     * tile — the entries the blend could composite; image, T, depth and
     * gradients are bit-identical to mode 0, n_contrib counts list entries. */
    int32_t bin_mode;
} lsb_settings;

/* World->camera rigid transform T_cw (SE3, geometry.py:125-171): p_c = R p_w + t.
 * R is row-major.  cam_center = -R^T t (raster.py:233) is passed explicitly so
 * host and device use the bit-identical value. */
typedef struct lsb_pose {
    double R[9];
    double t[3];
    double cam_center[3];
} lsb_pose;

/* Window parameter arena, structure-of-arrays (window.py:45-60):
 * means (n,3), rots (n,9) row-major 3x3, scales (n,3), opacities (n),
 * shs (n,K,3).  Device pointers.  dtype 0: f32 (the window arena's storage
 * type); dtype 1: f64 (the working copy optimize_window steps,
 * optimize.py:142-149, written back to f32 at the end). */
typedef struct lsb_params {
    const void* means;
    const void* rots;
    const void* scales;
    const void* opacities;
    const void* shs;
    int64_t n;
    int32_t sh_coeffs;   /* K = (degree+1)^2 stored per Gaussian */
    int32_t dtype;       /* 0 = f32, 1 = f64 */
} lsb_params;

/* Gradient buffers, same shapes as lsb_params but rot is the (n,3) right
 * tangent (ParamGradients, raster.py:85-98).  Backward ACCUMULATES (+=) into
 * them, so multi-view gradients sum without extra passes. */
typedef struct lsb_grads {
    float* mean;
    float* rot;
    float* scale;
    float* opacity;
    float* sh;
} lsb_grads;

/* Sizes that fix the workspace layout of one render state. */
typedef struct lsb_dims {
    int64_t n;            /* Gaussians                                  */
    int32_t width, height;
    int32_t sh_coeffs;
    int32_t tile;         /* must be 16                                 */
    int64_t isect_cap;    /* capacity for (tile, splat) intersections   */
} lsb_dims;

/* ---- size queries / diagnostics ------------------------------------- */
int lsb_abi_version(void);
const char* lsb_last_error(void);
int lsb_workspace_bytes(const lsb_dims* dims, size_t* bytes);

/* ---- render: replaces raster.render (raster.py:212-264) ---------------
 * Preprocess (projection, EWA covariance, footprint, SH colour; raster.py:
 * 134-185, 232-238), tile binning + per-tile depth sort (replaces the global
 * argsort + build_csr, raster.py:221, _kernels.py:21-59) and the front-to-back
 * blend (_kernels.py:62-119).  Outputs: image (H,W,3) f32, t_final (H,W) f32,
 * n_contrib (H,W) i32 and, if non-NULL, depth (H,W) f32 = sum_k w_k z_k.
 * The workspace then holds the render state consumed by lsb_render_bwd and
 * lsb_pose_rows.  If the intersection count exceeds dims->isect_cap the
 * outputs are invalid and lsb_render_counts reports overflow. */
int lsb_render_fwd(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw,
                   const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                   float* image, float* t_final, int32_t* n_contrib, float* depth,
                   void* stream);

/* ---- splat: replaces raster.splat (raster.py:188-205), batched --------
 * Per Gaussian i of p (async, device outputs): geo[7 i ..] = visible (1/0),
 * mu_i (x, y), cov_i (00, 01, 11), camera depth; color[3 i ..] = the
 * clipped SH colour (raster.py:232-238), valid where visible.  Same f64
 * projection / EWA covariance / footprint cull as the render's preprocess. */
int lsb_splat(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw, const lsb_settings* s,
              double* geo, double* color, void* stream);

/* ---- device sort / grouping (voxmap.py:213-230 group_by_leaf, window.py
 * and initialize.py key grouping) -------------------------------------------
 * Stable LSD radix sort of n (u64 key, i32 value) pairs on the low key_bits
 * bits (8-bit digits); vals_in NULL sorts the indices 0..n-1 along.  Outputs
 * must not alias the inputs.  lsb_segments: the start index of every run of
 * equal keys of a sorted array (starts: up to n entries; *nseg device int64).
 * Both use a caller workspace of lsb_sort_temp_bytes(n) bytes; async. */
int lsb_sort_temp_bytes(int64_t n, size_t* bytes);
int lsb_sort_pairs(const uint64_t* keys_in, const int32_t* vals_in, uint64_t* keys_out, int32_t* vals_out,
                   int64_t n, int key_bits, void* temp, size_t temp_bytes, void* stream);
int lsb_segments(const uint64_t* keys_sorted, int64_t n, int64_t* starts, int64_t* nseg, void* temp,
                 size_t temp_bytes, void* stream);

/* Synchronises `stream`; counts[0]=visible splats M, [1]=intersections I,
 * [2]=overflow flag (1 if I > isect_cap), [3]=isect_cap. */
int lsb_render_counts(const void* ws, const lsb_dims* dims, int64_t counts[4], void* stream);

/* Sticky capacity overflow of a workspace: set by every render whose
 * intersections exceed isect_cap (the per-render flag, counts[2], is reset
 * by the next render; this one is not).  `out` (host, may be NULL) receives
 * it after synchronising `stream`; clear != 0 then resets it (stream-ordered,
 * graph-capturable when out == NULL).  Call with clear = 1 once after
 * allocating a workspace. */
int lsb_render_sticky(void* ws, const lsb_dims* dims, int64_t* out, int clear, void* stream);

/* Synchronises `stream`; the alpha_cut band statistics of the last forward
 * (_kernels.py:104 decided in f64 where the blend's f32 alpha is within
 * CUT_BAND of the cut): out[0]=tiles re-blended, [1]=band pairs decided in
 * f64, [2]=of those, pairs composited, [3]=the largest relative error of the
 * f32 alpha against the f64 one over those pairs, as float bits.  All zero
 * when alpha_cut == 0. */
int lsb_render_band_stats(const void* ws, const lsb_dims* dims, int64_t out[4], void* stream);

/* Export the render state for parity checks (async):
 *   what=0: visible Gaussian ids, ascending (= slot order)  -> int32[M]
 *   what=1: bboxes [x0,x1,y0,y1] in slot order               -> int32[M*4]
 *   what=2: per-tile ranges [start,end)                      -> int32[ntiles*2]
 *   what=3: Gaussian id of every sorted tile entry           -> int32[I]
 *   what=4: camera depth (f64 sort key) in slot order        -> double[M]
 * M and I must come from lsb_render_counts. */
int lsb_render_export(const void* ws, const lsb_dims* dims, int what, void* dst, void* stream);

/* ---- backward: replaces raster.backward (raster.py:309-399) ----------
 * grad_image (H,W,3) f32 = dL/dI, multiplied by grad_scale.  Param
 * gradients are ACCUMULATED into `g`.  pose_out (device, 9 doubles) receives
 * the camera-tangent pose pieces [rho_cam(3), tau_cam(3), d_cam_center(3)];
 * the host applies -R d_cam_center and the IMU adjoint (raster.py:376-383). */
int lsb_render_bwd(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw,
                   const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                   const float* image, const float* t_final, const int32_t* n_contrib,
                   const float* grad_image, float grad_scale, const lsb_grads* g,
                   double* pose_out, void* stream);

/* ---- split launches of the same passes (for per-kernel timing / overlap) --
 * lsb_render_fwd == lsb_render_bin + lsb_render_blend;
 * lsb_render_bwd == lsb_render_blend_bwd + lsb_render_chain.            */
int lsb_render_bin(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw,
                   const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                   void* stream);
/* lsb_render_blend / lsb_render_blend_loss accept n_contrib == NULL (with
 * depth == NULL): no processed-entry count is kept, and the forward skips
 * half-tiles none of whose pixels reaches alpha_cut (same image / T bits).
 * lsb_render_blend_bwd does not read n_contrib (liveness is recomputed from
 * T bit-identically); it may be NULL. */
int lsb_render_blend(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                     float* image, float* t_final, int32_t* n_contrib, float* depth, void* stream);
/* Observed frames.  Every call taking `observed` with a loss `kind` (0 = L1,
 * 1 = L2) reads a float32 (H,W,3) image; with kind | LSB_OBS_U8 it reads the
 * camera's 8-bit (H,W,3) frame instead and uses u / 255.0 (f64), exactly the
 * reference's read_ppm (raster.py:520-541; dataset.py:231) — a quarter of
 * the host->device bytes, and the loss is formed from the same f64 values
 * the reference subtracts. */
#define LSB_OBS_U8 0x100

/* Blend forward fused with the photometric loss (optimize.py:48-74, no mask):
 * also writes grad_out (H,W,3) = dL/dI * grad_scale from observed (H,W,3) and
 * loss_out[0..1] = [sum |diff| (L1) or diff^2 (L2), sum diff^2] over all
 * pixels (deterministic: per-tile partials summed in tile order). */
int lsb_render_blend_loss(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                          float* image, float* t_final, int32_t* n_contrib, float* depth,
                          const void* observed, int kind, float grad_scale, float* grad_out,
                          double* loss_out, void* stream);
int lsb_render_blend_bwd(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                         const float* image, const int32_t* n_contrib, const float* grad_image,
                         float grad_scale, void* stream);
/* Blend backward with the photometric loss fused in (optimize.py:48-74, no
 * mask): dL/dI = sign(I - observed) (L1) or 2 (I - observed) (L2), times
 * grad_scale, is formed per pixel from image (the forward's output) and
 * observed (H,W,3), back-propagated like lsb_render_blend_bwd, and
 * loss_out[0..1] = [sum |diff| (L1) or diff^2 (L2), sum diff^2] (tile
 * partials summed in tile order; deterministic).  The window engine's step:
 * lsb_render_bin, lsb_render_blend (n_contrib NULL), this, lsb_render_chain. */
/* Forward + photometric loss + backward in one kernel (the window engine's
 * step after lsb_render_bin): the same results as lsb_render_blend (no
 * count) followed by lsb_render_blend_bwd_loss, without writing the image,
 * T or dL/dI; loss_out as there. */
int lsb_render_blend_fused_loss(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                                const void* observed, int kind, float grad_scale, double* loss_out, void* stream);
int lsb_render_blend_bwd_loss(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                              const float* image, const void* observed, int kind, float grad_scale,
                              double* loss_out, void* stream);
int lsb_render_chain(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw,
                     const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                     const lsb_grads* g, double* pose_out, void* stream);

/* ---- Adam in storage coordinates: replaces AdamState.update + the
 * optimize_window parameter steps (optimize.py:103-119, 159-188).
 * Updates the parameters IN PLACE through p (means, rots, scales,
 * opacities, shs; f32 or f64 per p->dtype).  grads is a flat f32 buffer
 * laid out [mean 3n | rot 3n | scale 3n | opacity n | sh 3Kn] (the
 * ParamGradients layout); m and v use the same layout in p->dtype;
 * touched (n bytes) records rotation rows that were stepped. */
typedef struct lsb_adam_cfg {
    double lr_mean, lr_rot, lr_scale, lr_opacity, lr_sh;
    double beta1, beta2, eps, scene_scale, opacity_clip, scale_floor;
    int64_t step;          /* 1-based shared step count (bias correction) */
} lsb_adam_cfg;
int lsb_adam_step(const lsb_params* p, const float* grads, void* m, void* v, uint8_t* touched,
                  const lsb_adam_cfg* cfg, void* stream);
/* The same step with the step count on the device, so a captured CUDA graph
 * can replay it: reads t = *step_dev + 1 (cfg->step is ignored), takes the
 * bias corrections from ibc_table[2(t-1)], ibc_table[2(t-1)+1] = 1/(1-beta1^t),
 * 1/(1-beta2^t) (host-computed like lsb_adam_step's; t beyond table_len uses
 * the last row), then increments *step_dev. */
int lsb_adam_step_dev(const lsb_params* p, const float* grads, void* m, void* v, uint8_t* touched,
                      const lsb_adam_cfg* cfg, const double* ibc_table, int64_t table_len, int64_t* step_dev,
                      void* stream);
/* Parameter groups of lsb_adam_step_dev_groups (gradient buffer ranges
 * [0,3n) mean, [3n,6n) rot, [6n,9n) scale, [9n,10n) opacity, [10n,..) sh). */
#define LSB_ADAM_MEAN 1
#define LSB_ADAM_ROT 2
#define LSB_ADAM_SCALE 4
#define LSB_ADAM_OPACITY 8
#define LSB_ADAM_SH 16
#define LSB_ADAM_ALL 31
/* lsb_adam_step_dev restricted to the parameter groups in `groups` (the
 * non-rotation groups must be contiguous in the order mean, scale, opacity,
 * sh), so a multi-GPU step can apply Adam to one all-reduce bucket while the
 * next bucket is still being reduced.  Every part of one step reads the same
 * step count t = *step_dev + 1; only the part with `advance` != 0 (the last
 * one) increments *step_dev.  The parts of a step together give the same
 * bits as one lsb_adam_step_dev call (each element's update is independent). */
int lsb_adam_step_dev_groups(const lsb_params* p, const float* grads, void* m, void* v, uint8_t* touched,
                             const lsb_adam_cfg* cfg, const double* ibc_table, int64_t table_len,
                             int64_t* step_dev, int32_t groups, int32_t advance, void* stream);
/* Fused multi-GPU optimiser step over NVLink peer memory (replaces the
 * NCCL all-reduce + Adam pair of the view-sharded step).  replicas[q] /
 * grads[q] / touched[q] are rank q's parameter arena, flat f32 gradient
 * buffer and touched flags as seen from this process (peer pointers, e.g.
 * from torch symmetric memory); n_ranks <= 8.  For the Gaussians [lo, hi)
 * this rank owns: gradients summed over ranks in rank order, Adam with this
 * rank's moments m / v, new parameters (and touched flags) stored into
 * EVERY replica.  The caller brackets the call with a cross-rank barrier.
 * ibc_table / step_dev as in lsb_adam_step_dev (both or neither). */
int lsb_adam_peer_step(const lsb_params* replicas, int32_t n_ranks, int32_t rank, const float* const* grads,
                       int64_t lo, int64_t hi, void* m, void* v, uint8_t* const* touched, const lsb_adam_cfg* cfg,
                       const double* ibc_table, int64_t table_len, int64_t* step_dev, void* stream);
/* Stage host bytes (pinned) into device memory on `stream` (observed
 * keyframe images each step; capturable into a CUDA graph). */
int lsb_copy_h2d(void* dst, const void* src, size_t bytes, void* stream);
/* Column Gram-Schmidt of touched rotation rows (optimize.py:91-100,193-194);
 * rots (n,9) in dtype (0 f32, 1 f64). */
int lsb_orthonormalize(void* rots, int32_t dtype, const uint8_t* touched, int64_t n, void* stream);

/* ---- pose rows + IESKF H/b: replaces raster.pose_rows (raster.py:402-508)
 * and the H^T R^-1 H / H^T R^-1 z products of ieskf_update
 * (estimator.py:278-280, 314-318) for the visual measurement.
 * lsb_pose_prepare writes LSB_POSE_CHAIN_FLOATS floats per visible splat
 * (L_mu, L_sig and the SH view-direction pieces) into `chain` (M rows, M
 * from lsb_render_counts).  lsb_pose_rows: one warp per selected pixel id
 * (flat row-major), rows_out (m,6) f64 = d gray(I_hat(u)) / d xi_IMU, using
 * the 6x6 row-major adjoint A (geometry.imu_camera_adjoint) and R_cw. */
#define LSB_POSE_CHAIN_FLOATS 48
int lsb_pose_prepare(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw,
                     const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* dims,
                     float* chain, void* stream);
int lsb_pose_rows(const lsb_settings* s, int sh_degree_used, void* ws, size_t ws_bytes,
                  const lsb_dims* dims, const float* image, const int32_t* n_contrib,
                  const float* chain, const int32_t* pixel_ids, int64_t m, const int64_t* m_dev,
                  const double* A, const double* R_cw, double* rows_out, void* stream);
/* m_dev (lsb_pose_rows, lsb_hb_reduce; may be NULL): a device count — only
 * the first min(*m_dev, m) ids / rows are used, so a count produced on the
 * device (lsb_visual_select's kept count, counts + 2) needs no host read.
 * out (42 doubles): [0..35] sum h h^T / sigma^2 (6x6), [36..41] sum h z / sigma^2,
 * h = -row (the pose block of H).  Deterministic: fixed-grid CTA partials in
 * `scratch` (lsb_hb_scratch_doubles() doubles), then a fixed-order sum. */
int lsb_hb_scratch_doubles(void);
int lsb_hb_reduce(const double* rows, const double* z, int64_t m, const int64_t* m_dev, double inv_sigma2,
                  double* out, double* scratch, void* stream);
/* One visual IESKF iteration in a single call (estimator.py:241-318 for the
 * pose block): lsb_render_fwd -> lsb_semidense_mask -> lsb_visual_select ->
 * lsb_pose_prepare -> lsb_pose_rows -> lsb_hb_reduce with the kept count on
 * the device, then the render's [M, I, overflow] counters copied next to
 * the selection counts.  Asynchronous; the caller reads b->out (48 x 8
 * bytes: int64 [L, selected, kept, M, I, overflow], then the 42 H/b
 * doubles) after one stream sync — the same bits as the separate calls. */
typedef struct lsb_visual_cfg {
    int32_t budget;             /* pixel_budget */
    int32_t observed_u8;        /* observed is the 8-bit frame */
    int32_t sh_degree_used;
    int32_t _pad;
    double grad_thr, t_max, gate, inv_sigma2;
    double A[36];               /* imu_camera_adjoint(R_cw, T_ic), row-major */
} lsb_visual_cfg;
typedef struct lsb_visual_bufs {
    uint8_t* mask;              /* H*W */
    void* select_scratch;       /* lsb_visual_select_scratch_bytes(H*W, budget) */
    int32_t* ids;               /* budget */
    double* res;                /* budget */
    float* chain;               /* n * LSB_POSE_CHAIN_FLOATS */
    double* rows;               /* budget * 6 */
    double* hb_scratch;         /* lsb_hb_scratch_doubles() */
    int64_t* out;               /* 48 x 8 bytes, see above */
} lsb_visual_bufs;
int lsb_visual_pass(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T_cw, const lsb_settings* s,
                    void* ws, size_t ws_bytes, const lsb_dims* dims, float* image, float* t_final,
                    int32_t* n_contrib, const void* observed, const lsb_visual_cfg* cfg, const lsb_visual_bufs* b,
                    void* stream);

/* Host-side gain algebra of one IESKF iteration for a pose-block measurement
 * (estimator.py:292-331): P = Hj^-1 cov Hj^-T (Hj^-1 = I with jinv3 =
 * J_l(-delta_rho) in the rotation block), S = A + P^-1 (A = the 6x6 block
 * A6), K H = S^-1 A -> KH (15x15), xi = -S^-1 b - (I - K H) Hj^-1 delta
 * (b = b6 padded) -> xi (15), P -> P (15x15).  All host pointers, row-major.
 * LSB_EINVAL with "singular matrix" / "non-finite gain" where the reference
 * raises SingularGain. */
int lsb_ieskf_gain(const double* cov, const double* jinv3, const double* A6, const double* b6, const double* delta,
                   double* xi, double* KH, double* P);

/* A whole IESKF iteration on the host state vectors x = [R (9, row-major) |
 * t | v | b_g | b_a] (21 doubles): delta = x_hat [-] x_bar (NavState.boxminus,
 * estimator.py:70-75), lsb_ieskf_gain, then x_hat <- x_hat [+] xi in place
 * (NavState.boxplus with the bias clip, estimator.py:63-68); xi, KH, P out as
 * in lsb_ieskf_gain. */
int lsb_ieskf_iterate(const double* cov, const double* x_bar, double* x_hat, const double* A6, const double* b6,
                      double bias_limit, double* xi, double* KH, double* P);

/* Semi-dense candidate mask (estimator.py:241-252): Sobel/8 magnitude of the
 * grey observed image (nearest border) > grad_thr and t_final < t_max.
 * observed_u8 (here and in lsb_visual_select): the frame is 8-bit, read as
 * u / 255.0 like LSB_OBS_U8; else float32. */
int lsb_semidense_mask(const void* observed, int32_t observed_u8, const float* t_final, int32_t width,
                       int32_t height, double grad_thr, double t_max, uint8_t* mask_out, void* stream);

/* Visual measurement selection, on the device with no host round trip
 * (estimator.py:241-277 after the render): from the semi-dense mask, the
 * candidate ids ascending, subsampled to `budget` at round(linspace(0, L-1,
 * budget)); the grey residual obs - image (channel means in f64) kept where
 * |res| <= gate, in order -> ids_out / res_out (budget entries max);
 * counts (device, 3 int64) = [candidates L, selected, kept].  scratch:
 * lsb_visual_select_scratch_bytes(npx, budget) bytes. */
int64_t lsb_visual_select_scratch_bytes(int64_t npx, int32_t budget);
int lsb_visual_select(const uint8_t* mask, const void* observed, int32_t observed_u8, const float* image, int64_t npx,
                      int32_t budget,
                      double gate, void* scratch, int32_t* ids_out, double* res_out, int64_t* counts, void* stream);

/* ---- voxel map: replaces HashOctree's batch operations (voxmap.py:99-251)
 * Open-addressing table of octree LEAVES (the octree is implied by its leaf
 * set; parents/roots by floor division).  All arrays are caller-allocated
 * device memory of `cap` entries (cap a power of two); keys start as
 * 0xFF..FF, count/sum/outer as 0, gslot as -1, claim as INT32_MAX.
 * Keys are floor(p / edge) in f64 with true division (voxmap.py:45-65). */
typedef struct lsb_voxmap {
    uint64_t* keys;          /* packed (ix, iy, iz), 21 bits each            */
    uint64_t* count;         /* points accumulated per leaf                 */
    double* sum;             /* (cap, 3) sum p                              */
    double* outer;           /* (cap, 6) sum p p^T: xx xy xz yy yz zz       */
    int32_t* gslot;          /* Gaussian id held by the leaf, -1 if none     */
    int32_t* claim;          /* try_insert scratch                          */
    uint64_t* n_used;        /* occupied slots (device counter)             */
    uint64_t* flags;         /* sticky error flag (table full / key range)  */
    int64_t cap;
    double root_len;
    int32_t max_level;
    int32_t _pad;
    uint64_t* gkeys;         /* (cap) packed keys of the leaves holding a Gaussian, append-only (may be
                                NULL: the FoV then scans the whole table)      */
    uint64_t* n_gkeys;       /* entries of gkeys (device counter)            */
} lsb_voxmap;
/* keys_of_points: (n,3) f64 points -> (n,3) int64 floor(p / edge). */
int lsb_voxmap_keys(const double* pts, int64_t n, double edge, int64_t* keys_out, void* stream);
/* accumulate_points: create the leaves containing pts and, if accumulate is
 * non-zero, add (count, sum, outer) (add_leaf_stats); accumulate == 0 is
 * ensure_leaf / locate_or_subdivide.  slots_out (n) int64 receives each
 * point's leaf slot (may be NULL). */
int lsb_voxmap_insert_points(const lsb_voxmap* m, const double* pts, int64_t n, int32_t accumulate,
                             int64_t* slots_out, void* stream);
/* Deterministic accumulate_points (voxmap.py:184-211): each leaf adds its
 * group's count / sum / outer once; the group sums are exact (per-point
 * terms in 128-bit fixed point, 2^-60, added with integer atomics, which
 * are order-free) and rounded to f64 once - identical statistics run to run
 * (lsb_voxmap_insert_points with accumulate uses f64 atomics instead).
 * Uses the map's claim scratch (restored).  temp:
 * lsb_voxmap_accumulate_temp_bytes(n) bytes. */
int lsb_voxmap_accumulate_temp_bytes(int64_t n, size_t* bytes);
int lsb_voxmap_accumulate(const lsb_voxmap* m, const double* pts, int64_t n, int64_t* slots_out, void* temp,
                          size_t temp_bytes, void* stream);
/* try_insert for a batch of Gaussian means with leaf_capacity 1: the lowest
 * batch index landing in an empty leaf is stored (gslot = first_gid + i) and
 * gets status 1 (Inserted), the others 0 (Full).  slots (n) int64 scratch. */
int lsb_voxmap_try_insert(const lsb_voxmap* m, const double* means, int64_t n, int32_t first_gid,
                          int64_t* slots, int32_t* status_out, void* stream);
/* get_leaf for (n,3) int64 leaf keys -> slot or -1. */
int lsb_voxmap_lookup(const lsb_voxmap* m, const int64_t* keys, int64_t n, int64_t* slots_out,
                      void* stream);
/* FoV leaves: leaves holding a Gaussian under the root voxels touched by
 * pts (leaf_keys_under_roots(keys_of_points(pts, root_len, 0))).  rset is a
 * caller scratch of rcap (power of two) u64; out (out_cap,3) int64 keys,
 * n_out (device u64) the count (may exceed out_cap: then grow and retry). */
int lsb_voxmap_fov(const lsb_voxmap* m, const double* pts, int64_t n, uint64_t* rset, int64_t rcap,
                   int64_t* out, uint64_t* n_out, int64_t out_cap, void* stream);
/* Occupied leaves -> (keys (k,3) int64, slots (k) int64), k in *n_out. */
int lsb_voxmap_dump(const lsb_voxmap* m, int64_t* keys, int64_t* slots, uint64_t* n_out,
                    int64_t out_cap, void* stream);
/* Re-insert every leaf of `src` into the (larger, empty) table `dst`. */
int lsb_voxmap_rehash(const lsb_voxmap* src, const lsb_voxmap* dst, void* stream);

/* Plane fits: replaces HashOctree.fit_planes / estimate_normal / plane_at
 * (voxmap.py:255-335).  Per leaf key (k,3): the leaf's and its 6 face
 * neighbours' statistics, the smallest-scatter eigenvector (f64 Jacobi)
 * facing `origin` and the leaf's own centroid; valid[i] = 0 (NaN rows) for
 * an empty leaf, fewer than 3 points or scatter rank < 2. */
int lsb_voxmap_fit_planes(const lsb_voxmap* m, const int64_t* keys, int64_t k, const double* origin, double* normals,
                          double* anchors, uint8_t* valid, void* stream);
/* LiDAR point-to-plane rows: replaces the per-point part of
 * lidar_measurement (estimator.py:190-238).  pts_l (n,3) f64 in the LiDAR
 * frame; T_IL and T_WI as row-major R and t.  Per point: rows (n,6) =
 * -H[:, :6] (the lsb_hb_reduce convention), z = n . (p_w - anchor),
 * keep = a plane was found for the point's leaf and |z| <= gate. */
int lsb_lidar_rows(const lsb_voxmap* m, const double* pts_l, int64_t n, const double* R_il, const double* t_il,
                   const double* R_wi, const double* t_wi, double gate, double* rows, double* z, uint8_t* keep,
                   void* stream);

/* Batched Gaussian initialisation: replaces the per-leaf loop of
 * pipeline._insert_new_gaussians + initialize.init_gaussian
 * (pipeline.py:99-137, initialize.py:22-124).  keys (k,3) the scan's leaf
 * groups in sorted order, centroids (k,3) f64 their scan centroids, image
 * (H,W,3) f32, T_CW row-major, cam4 = fx fy cx cy, origin = the sensor
 * position.  rows (k, 16+3K) f32 (the arena row layout) and status[i] = 1
 * where a Gaussian was made (leaf empty, observable, in the image
 * interior); the caller stores those rows in the map. */
int lsb_init_gaussians(const lsb_voxmap* m, const int64_t* keys, const double* centroids, int64_t k,
                       const float* image, int32_t width, int32_t height, const double* R_cw, const double* t_cw,
                       const double* cam4, const double* origin, double near, double kappa, double delta,
                       double opacity, int32_t sh_coeffs, float* rows, uint8_t* status, void* stream);

/* Group means (group_by_leaf + points.mean(axis=0), voxmap.py:213-230,
 * pipeline.py:113): group g is points perm[starts[g] .. starts[g]+counts[g])
 * in that order; out (k,3) f64 = their sum, row by row, / count. */
int lsb_segment_mean(const double* pts, const int64_t* perm, const int64_t* starts, const int64_t* counts, int64_t k,
                     double* out, void* stream);

/* ---- sliding window: replaces GaussianWindow.maintain (window.py:136-276)
 * The live window is the f32 SoA arena `arena` (capacity rows, n live); the
 * global map's Gaussians are rows of `store` (mean 3 | rot 9 | scale 3 |
 * opacity 1 | sh 3K floats, the reference's arena row, window.py:58-60)
 * indexed by the leaf's gid (lsb_voxmap.gslot).  Keys are "order keys"
 * ((ix+2^20) << 42 | (iy+2^20) << 21 | (iz+2^20)): integer order is sorted
 * VoxelKey order.  wkeys (capacity) holds the key of every slot, -1 if free.
 *   mark:    rebuild the window hash (hkeys/hslots, hcap a power of two >=
 *            2n) and probe the m FoV keys: keep[slot] = 1 for live ∩ FoV,
 *            is_add[i] = 1 for FoV keys not live (diff, window.py:136-143).
 *   plan:    one CTA: dels = deleted slots ascending, movers = the live slots
 *            at or above the new live count, from the rear; counts = [k, h]
 *            (deleted, moves).  Synchronise to read counts.
 *   compact: write the k deleted rows back to the map store (their leaves'
 *            gids; flag bit 2 on a missing leaf), then move movers[r] ->
 *            dels[r] for r < h and free the top k slots (window.py:145-181).
 *   leaf_gids / dist: per (sorted) add key, the map gid (-1: no Gaussian) and
 *            the f64 distance of the voxel centre to `origin` (numpy's
 *            norm, for the capacity ranking, window.py:262-270).
 *   append:  the adds holding a Gaussian, in key order, to slots first_slot,
 *            first_slot + 1, ... (*n_added on the device; window.py:183-209). */
int lsb_window_mark(const int64_t* wkeys, int64_t n, uint64_t* hkeys, int32_t* hslots, int64_t hcap,
                    const int64_t* fov, int64_t m, uint8_t* keep, uint8_t* is_add, void* stream);
/* plan / append take an int32 scratch of lsb_window_plan_tiles(n) /
 * lsb_window_append_tiles(cnt) entries (per-tile counts and offsets). */
int64_t lsb_window_plan_tiles(int64_t n);
int64_t lsb_window_append_tiles(int64_t cnt);
int lsb_window_plan(const uint8_t* keep, int64_t n, int32_t* dels, int32_t* movers, int64_t* counts, int32_t* tiles,
                    void* stream);
int lsb_window_compact(const lsb_voxmap* m, const lsb_params* arena, int64_t* wkeys, const int32_t* dels, int64_t k,
                       const int32_t* movers, int64_t h, int64_t n, float* store, void* stream);
int lsb_window_leaf_gids(const lsb_voxmap* m, const int64_t* okeys, int64_t cnt, int32_t* gids, void* stream);
int lsb_window_dist(const int64_t* okeys, int64_t cnt, double edge, const double* origin, double* out,
                    void* stream);
int lsb_window_append(const lsb_params* arena, int64_t* wkeys, const int64_t* okeys, const int32_t* gids, int64_t cnt,
                      const float* store, int64_t first_slot, int64_t* n_added, int32_t* tiles, void* stream);

/* ---- photometric loss: replaces optimize.photometric_loss (optimize.py:48-74)
 * kind 0 = L1, 1 = L2 over (npx, 3) f32 images; mask (npx) u8 may be NULL.
 * grad_out (npx,3) f32 = sign(diff) (L1) or 2 diff (L2), times grad_scale
 * (the host passes 1/(3*mask_count) [/ views]); may be NULL.
 * sums_out: device buffer of lsb_loss_scratch_doubles() doubles, zeroed once
 * at allocation; on completion sums_out[0] = sum |diff| (L1) or sum diff^2
 * (L2) and sums_out[1] = sum diff^2 over the mask.  Deterministic. */
int lsb_loss_scratch_doubles(void);
int lsb_photometric_loss(const float* rendered, const void* observed, const uint8_t* mask,
                         int64_t npx, int64_t mask_count, int kind, float grad_scale,
                         float* grad_out, double* sums_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSB_H */
