// extern "C" entry points of libsplat_b200.so (declared in include/lsb.h).
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace lsb {
cudaError_t launch_splat(const lsb_params&, const lsb_camera&, const lsb_pose&, const lsb_settings&, double*, double*,
                         cudaStream_t);
size_t sort_temp_bytes(int64_t n);
cudaError_t launch_sort_pairs(const uint64_t*, const int32_t*, uint64_t*, int32_t*, int64_t, int, void*, cudaStream_t);
cudaError_t launch_segments(const uint64_t*, int64_t, int64_t*, int64_t*, void*, cudaStream_t);
size_t vox_accumulate_temp_bytes(int64_t n);
cudaError_t launch_vox_accumulate(const lsb_voxmap&, const double*, int64_t, int64_t*, void*, cudaStream_t);
cudaError_t launch_preprocess(const lsb_params&, const lsb_camera&, const lsb_pose&, const lsb_settings&,
                              const Ws&, cudaStream_t);
cudaError_t launch_blend_fwd(const Ws&, const lsb_settings&, int, int, float*, float*, int32_t*, float*,
                             const void*, int, float, float*, double*, cudaStream_t);
cudaError_t launch_blend_fused(const Ws&, const lsb_settings&, int, int, const void*, int, float, double*, cudaStream_t);
cudaError_t launch_blend_bwd_loss(const Ws&, const lsb_settings&, int, int, const float*, const void*, int, float,
                                  double*, cudaStream_t);
cudaError_t launch_blend_bwd(const Ws&, const lsb_settings&, int, int, const float*, const int32_t*,
                             const float*, float, cudaStream_t);
cudaError_t launch_chain(const Ws&, const lsb_params&, const lsb_grads&, const lsb_camera&, const lsb_pose&,
                         const lsb_settings&, double*, cudaStream_t);
cudaError_t launch_loss(const float*, const void*, const uint8_t*, int64_t, int, float, float*, double*,
                        cudaStream_t);
int loss_scratch_doubles();
cudaError_t launch_adam(const lsb_params&, const float*, void*, void*, uint8_t*, const lsb_adam_cfg&, const double*,
                        int64_t, int64_t*, cudaStream_t, int groups = LSB_ADAM_ALL, bool advance = true);
bool adam_groups_contiguous(int groups);
cudaError_t launch_orthonormalize(void*, int, const uint8_t*, int64_t, cudaStream_t);
cudaError_t launch_adam_peer(const lsb_params*, int, int, const float* const*, int64_t, int64_t, void*, void*,
                             uint8_t* const*, const lsb_adam_cfg&, const double*, int64_t, int64_t*, cudaStream_t);
int adam_max_peers();
cudaError_t launch_pose_prepare(const Ws&, const lsb_params&, const lsb_camera&, const lsb_pose&,
                                const lsb_settings&, float*, cudaStream_t);
cudaError_t launch_pose_rows(const Ws&, const lsb_settings&, int, int, int, const float*, const int32_t*,
                             const float*, const int32_t*, int64_t, const int64_t*, const double*, const double*,
                             double*, cudaStream_t);
cudaError_t launch_hb(const double*, const double*, int64_t, const int64_t*, double, double*, double*, cudaStream_t);
int hb_scratch_doubles();
int ieskf_gain(const double*, const double*, const double*, const double*, const double*, double*, double*, double*);
int ieskf_iterate(const double*, const double*, double*, const double*, const double*, double, double*, double*,
                  double*);
cudaError_t launch_visual_select(const uint8_t*, const void*, bool, const float*, int64_t, int, double, void*, int32_t*,
                                 double*, int64_t*, cudaStream_t);
int64_t visual_select_scratch_bytes(int64_t, int);
cudaError_t launch_semidense(const void*, bool, const float*, int, int, double, double, uint8_t*, cudaStream_t);
cudaError_t launch_vox_keys(const double*, int64_t, double, int64_t*, cudaStream_t);
cudaError_t launch_vox_insert(const lsb_voxmap&, const double*, int64_t, int, int64_t*, cudaStream_t);
cudaError_t launch_vox_try_insert(const lsb_voxmap&, const double*, int64_t, int32_t, int64_t*, int32_t*,
                                  cudaStream_t);
cudaError_t launch_vox_lookup(const lsb_voxmap&, const int64_t*, int64_t, int64_t*, cudaStream_t);
cudaError_t launch_vox_fov(const lsb_voxmap&, const double*, int64_t, unsigned long long*, int64_t, int64_t*,
                           unsigned long long*, int64_t, cudaStream_t);
cudaError_t launch_vox_dump(const lsb_voxmap&, int64_t*, int64_t*, unsigned long long*, int64_t, cudaStream_t);
cudaError_t launch_vox_rehash(const lsb_voxmap&, const lsb_voxmap&, cudaStream_t);
cudaError_t launch_fit_planes(const lsb_voxmap&, const int64_t*, int64_t, const double*, double*, double*, uint8_t*,
                              cudaStream_t);
cudaError_t launch_lidar_rows(const lsb_voxmap&, const double*, int64_t, const double*, const double*, const double*,
                              const double*, double, double, double*, double*, uint8_t*, cudaStream_t);
cudaError_t launch_init_gaussians(const lsb_voxmap&, const int64_t*, const double*, int64_t, const float*, int, int,
                                  const double*, const double*, const double*, const double*, double, double, double,
                                  double, int, float*, uint8_t*, cudaStream_t);
cudaError_t launch_segment_mean(const double*, const int64_t*, const int64_t*, const int64_t*, int64_t, double*,
                                cudaStream_t);
cudaError_t launch_win_mark(const int64_t*, int64_t, uint64_t*, int32_t*, int64_t, const int64_t*, int64_t, uint8_t*,
                            uint8_t*, cudaStream_t);
cudaError_t launch_win_plan(const uint8_t*, int64_t, int32_t*, int32_t*, int64_t*, int32_t*, cudaStream_t);
int64_t win_plan_tiles(int64_t);
int64_t win_append_tiles(int64_t);
cudaError_t launch_win_compact(const lsb_voxmap&, const lsb_params&, int64_t*, const int32_t*, int64_t,
                               const int32_t*, int64_t, int64_t, float*, cudaStream_t);
cudaError_t launch_win_leaf_gids(const lsb_voxmap&, const int64_t*, int64_t, int32_t*, cudaStream_t);
cudaError_t launch_win_dist(const int64_t*, int64_t, double, const double*, double*, cudaStream_t);
cudaError_t launch_win_append(const lsb_params&, int64_t*, const int64_t*, const int32_t*, int64_t, const float*,
                              int64_t, int64_t*, int32_t*, cudaStream_t);
}  // namespace lsb

using namespace lsb;

static thread_local char g_err[512] = "";

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

static int check_cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return LSB_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return LSB_ECUDA;
}

static int dims_ok(const lsb_dims* d) {
    if (!d) return fail(LSB_EINVAL, "dims is NULL");
    if (d->n < 0 || d->width <= 0 || d->height <= 0) return fail(LSB_EINVAL, "bad dims");
    if (d->width > 32767 || d->height > 32767) return fail(LSB_EINVAL, "image larger than 32767 px");
    if (d->tile != TILE) return fail(LSB_EINVAL, "tile must be 16");
    if (d->isect_cap < 1 || d->isect_cap > 0x7fffffffLL) return fail(LSB_EINVAL, "bad isect_cap");
    if (d->n > 0x7fffffffLL) return fail(LSB_EINVAL, "too many Gaussians for int32 ids");
    return LSB_OK;
}

static int get_ws(void* ws, size_t ws_bytes, const lsb_dims* d, Ws* w) {
    int rc = dims_ok(d);
    if (rc) return rc;
    if (!ws) return fail(LSB_EMISSING_CACHE, "workspace is NULL (render state missing)");
    const size_t need = carve(*d, nullptr, nullptr);
    if (ws_bytes < need) return fail(LSB_EINVAL, "workspace too small");
    carve(*d, (char*)ws, w);
    return LSB_OK;
}

extern "C" {

int lsb_abi_version(void) { return LSB_ABI_VERSION; }

const char* lsb_last_error(void) { return g_err; }

int lsb_workspace_bytes(const lsb_dims* d, size_t* bytes) {
    int rc = dims_ok(d);
    if (rc) return rc;
    if (!bytes) return fail(LSB_EINVAL, "bytes is NULL");
    *bytes = carve(*d, nullptr, nullptr);
    return LSB_OK;
}

int lsb_loss_scratch_doubles(void) { return loss_scratch_doubles(); }

int lsb_render_fwd(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s,
                   void* ws, size_t ws_bytes, const lsb_dims* d, float* image, float* t_final,
                   int32_t* n_contrib, float* depth, void* stream) {
    if (!p || !cam || !T || !s) return fail(LSB_EINVAL, "NULL argument");
    if (!image || !t_final || !n_contrib) return fail(LSB_EINVAL, "NULL output");
    if (p->n != d->n || cam->width != d->width || cam->height != d->height)
        return fail(LSB_EINVAL, "dims do not match params/camera");
    if (p->n > 0 && (!p->means || !p->rots || !p->scales || !p->opacities || !p->shs))
        return fail(LSB_EINVAL, "NULL parameter array");
    if (p->sh_coeffs < 1 || p->sh_coeffs > 16) return fail(LSB_EINVAL, "sh_coeffs must be 1..16");
    if (p->dtype != 0 && p->dtype != 1) return fail(LSB_EINVAL, "params dtype must be 0 (f32) or 1 (f64)");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    rc = check_cuda(launch_preprocess(*p, *cam, *T, *s, w, st), "preprocess");
    if (rc) return rc;
    return check_cuda(launch_blend_fwd(w, *s, d->width, d->height, image, t_final, n_contrib, depth, nullptr, 0, 0.f, nullptr,
                                       nullptr, st),
                      "blend_fwd");
}

int lsb_sort_temp_bytes(int64_t n, size_t* bytes) {
    if (!bytes || n < 0) return fail(LSB_EINVAL, "bad argument");
    *bytes = sort_temp_bytes(n);
    return LSB_OK;
}

int lsb_sort_pairs(const uint64_t* keys_in, const int32_t* vals_in, uint64_t* keys_out, int32_t* vals_out, int64_t n,
                   int key_bits, void* temp, size_t temp_bytes, void* stream) {
    if (n < 0 || n > 0x7fffffffll || key_bits < 1 || key_bits > 64) return fail(LSB_EINVAL, "bad n or key_bits");
    if (n > 0 && (!keys_in || !keys_out || !vals_out || !temp)) return fail(LSB_EINVAL, "NULL argument");
    if ((const void*)keys_in == (const void*)keys_out || (vals_in && (const void*)vals_in == (const void*)vals_out))
        return fail(LSB_EINVAL, "sort outputs must not alias the inputs");
    if (temp_bytes < sort_temp_bytes(n)) return fail(LSB_EINVAL, "sort workspace too small");
    return check_cuda(launch_sort_pairs(keys_in, vals_in, keys_out, vals_out, n, key_bits, temp, (cudaStream_t)stream),
                      "sort_pairs");
}

int lsb_segments(const uint64_t* keys_sorted, int64_t n, int64_t* starts, int64_t* nseg, void* temp,
                 size_t temp_bytes, void* stream) {
    if (n < 0 || n > 0x7fffffffll) return fail(LSB_EINVAL, "bad n");
    if (!nseg || (n > 0 && (!keys_sorted || !starts || !temp))) return fail(LSB_EINVAL, "NULL argument");
    if (temp_bytes < sort_temp_bytes(n)) return fail(LSB_EINVAL, "sort workspace too small");
    return check_cuda(launch_segments(keys_sorted, n, starts, nseg, temp, (cudaStream_t)stream), "segments");
}

int lsb_splat(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s, double* geo,
              double* color, void* stream) {
    if (!p || !cam || !T || !s || !geo || !color) return fail(LSB_EINVAL, "NULL argument");
    if (p->n > 0 && (!p->means || !p->rots || !p->scales || !p->opacities || !p->shs))
        return fail(LSB_EINVAL, "NULL parameter array");
    if (p->sh_coeffs < 1 || p->sh_coeffs > 16) return fail(LSB_EINVAL, "sh_coeffs must be 1..16");
    if (p->dtype != 0 && p->dtype != 1) return fail(LSB_EINVAL, "params dtype must be 0 (f32) or 1 (f64)");
    return check_cuda(launch_splat(*p, *cam, *T, *s, geo, color, (cudaStream_t)stream), "splat");
}

int lsb_render_counts(const void* ws, const lsb_dims* d, int64_t counts[4], void* stream) {
    Ws w;
    int rc = get_ws((void*)ws, (size_t)-1, d, &w);
    if (rc) return rc;
    unsigned long long h[3];
    cudaStream_t st = (cudaStream_t)stream;
    rc = check_cuda(cudaMemcpyAsync(h, w.ctr, sizeof(h), cudaMemcpyDeviceToHost, st), "counts");
    if (rc) return rc;
    rc = check_cuda(cudaStreamSynchronize(st), "counts sync");
    if (rc) return rc;
    counts[0] = (int64_t)h[0];
    counts[1] = (int64_t)h[1];
    counts[2] = (int64_t)h[2];
    counts[3] = d->isect_cap;
    return LSB_OK;
}

int lsb_render_sticky(void* ws, const lsb_dims* d, int64_t* out, int clear, void* stream) {
    Ws w;
    int rc = get_ws(ws, (size_t)-1, d, &w);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (out) {
        unsigned long long h = 0;
        rc = check_cuda(cudaMemcpyAsync(&h, w.sticky, sizeof(h), cudaMemcpyDeviceToHost, st), "sticky");
        if (rc) return rc;
        rc = check_cuda(cudaStreamSynchronize(st), "sticky sync");
        if (rc) return rc;
        *out = (int64_t)h;
    }
    if (clear) return check_cuda(cudaMemsetAsync(w.sticky, 0, sizeof(unsigned long long), st), "sticky clear");
    return LSB_OK;
}

int lsb_render_band_stats(const void* ws, const lsb_dims* d, int64_t out[4], void* stream) {
    Ws w;
    int rc = get_ws((void*)ws, (size_t)-1, d, &w);
    if (rc) return rc;
    unsigned long long h[16];
    cudaStream_t st = (cudaStream_t)stream;
    rc = check_cuda(cudaMemcpyAsync(h, w.ctr, sizeof(h), cudaMemcpyDeviceToHost, st), "band stats");
    if (rc) return rc;
    rc = check_cuda(cudaStreamSynchronize(st), "band stats sync");
    if (rc) return rc;
    out[0] = (int64_t)h[9];
    out[1] = (int64_t)h[12];
    out[2] = (int64_t)h[13];
    out[3] = (int64_t)(h[14] & 0xffffffffull);
    return LSB_OK;
}

namespace lsb {
__global__ void k_export(Ws w, int what, void* dst) {
    const int64_t M = (int64_t)w.ctr[0];
    const int64_t I = (int64_t)w.ctr[1];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (what == 0) {
        for (int64_t i = i0; i < M; i += stride) ((int32_t*)dst)[i] = w.rec[i].id;
    } else if (what == 1) {
        for (int64_t i = i0; i < M; i += stride) {
            const Rec& r = w.rec[i];
            int32_t* o = (int32_t*)dst + 4 * i;
            o[0] = r.bbx & 0xffff; o[1] = r.bbx >> 16; o[2] = r.bby & 0xffff; o[3] = r.bby >> 16;
        }
    } else if (what == 2) {
        for (int64_t t = i0; t < w.ntiles; t += stride) {
            ((int32_t*)dst)[2 * t] = w.tile_start[t];
            ((int32_t*)dst)[2 * t + 1] = w.tile_start[t + 1];
        }
    } else if (what == 3) {
        for (int64_t j = i0; j < I && j < w.cap; j += stride) ((int32_t*)dst)[j] = w.rec[w.tile_slot[j] & SLOT_MASK].id;
    } else if (what == 4) {
        for (int64_t i = i0; i < M; i += stride) ((double*)dst)[i] = __longlong_as_double((long long)w.vkey[i]);
    }
}
}  // namespace lsb

int lsb_render_export(const void* ws, const lsb_dims* d, int what, void* dst, void* stream) {
    Ws w;
    int rc = get_ws((void*)ws, (size_t)-1, d, &w);
    if (rc) return rc;
    if (!dst || what < 0 || what > 4) return fail(LSB_EINVAL, "bad export request");
    k_export<<<148, 256, 0, (cudaStream_t)stream>>>(w, what, dst);
    return check_cuda(cudaGetLastError(), "export");
}

int lsb_render_bwd(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s,
                   void* ws, size_t ws_bytes, const lsb_dims* d, const float* image,
                   const float* t_final, const int32_t* n_contrib, const float* grad_image,
                   float grad_scale, const lsb_grads* g, double* pose_out, void* stream) {
    (void)t_final;
    if (!p || !cam || !T || !s || !g) return fail(LSB_EINVAL, "NULL argument");
    if (!image || !n_contrib || !grad_image) return fail(LSB_EMISSING_CACHE, "render outputs missing");
    if (p->n > 0 && (!g->mean || !g->rot || !g->scale || !g->opacity || !g->sh))
        return fail(LSB_EINVAL, "NULL gradient array");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    rc = check_cuda(launch_blend_bwd(w, *s, d->width, d->height, image, n_contrib, grad_image, grad_scale, st),
                    "blend_bwd");
    if (rc) return rc;
    return check_cuda(launch_chain(w, *p, *g, *cam, *T, *s, pose_out, st), "chain");
}

static int params_ok(const lsb_params* p, const lsb_dims* d) {
    if (!p) return fail(LSB_EINVAL, "NULL params");
    if (p->n != d->n) return fail(LSB_EINVAL, "dims do not match params");
    if (p->n > 0 && (!p->means || !p->rots || !p->scales || !p->opacities || !p->shs))
        return fail(LSB_EINVAL, "NULL parameter array");
    if (p->sh_coeffs < 1 || p->sh_coeffs > 16) return fail(LSB_EINVAL, "sh_coeffs must be 1..16");
    if (p->dtype != 0 && p->dtype != 1) return fail(LSB_EINVAL, "params dtype must be 0 (f32) or 1 (f64)");
    return LSB_OK;
}

int lsb_render_bin(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s,
                   void* ws, size_t ws_bytes, const lsb_dims* d, void* stream) {
    if (!cam || !T || !s) return fail(LSB_EINVAL, "NULL argument");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    rc = params_ok(p, d);
    if (rc) return rc;
    if (cam->width != d->width || cam->height != d->height) return fail(LSB_EINVAL, "camera/dims mismatch");
    return check_cuda(launch_preprocess(*p, *cam, *T, *s, w, (cudaStream_t)stream), "bin");
}

int lsb_render_blend(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* d, float* image,
                     float* t_final, int32_t* n_contrib, float* depth, void* stream) {
    if (!s || !image || !t_final) return fail(LSB_EINVAL, "NULL argument");
    if (!n_contrib && depth) return fail(LSB_EINVAL, "depth needs n_contrib");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    return check_cuda(launch_blend_fwd(w, *s, d->width, d->height, image, t_final, n_contrib, depth, nullptr, 0,
                                       0.f, nullptr, nullptr, (cudaStream_t)stream), "blend");
}

int lsb_render_blend_loss(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* d, float* image,
                          float* t_final, int32_t* n_contrib, float* depth, const void* observed, int kind,
                          float grad_scale, float* grad_out, double* loss_out, void* stream) {
    if (!s || !image || !t_final || !observed || !grad_out || !loss_out)
        return fail(LSB_EINVAL, "NULL argument");
    if (!n_contrib && depth) return fail(LSB_EINVAL, "depth needs n_contrib");
    if ((kind & ~LSB_OBS_U8) != 0 && (kind & ~LSB_OBS_U8) != 1)
        return fail(LSB_EINVAL, "kind must be 0 (l1) or 1 (l2), optionally | LSB_OBS_U8");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    return check_cuda(launch_blend_fwd(w, *s, d->width, d->height, image, t_final, n_contrib, depth, observed,
                                       kind, grad_scale, grad_out, loss_out, (cudaStream_t)stream),
                      "blend_loss");
}

int lsb_render_blend_bwd(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* d,
                         const float* image, const int32_t* n_contrib, const float* grad_image,
                         float grad_scale, void* stream) {
    if (!s) return fail(LSB_EINVAL, "NULL argument");
    if (!image || !grad_image) return fail(LSB_EMISSING_CACHE, "render outputs missing");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    return check_cuda(launch_blend_bwd(w, *s, d->width, d->height, image, n_contrib, grad_image, grad_scale,
                                       (cudaStream_t)stream), "blend_bwd");
}

int lsb_render_blend_fused_loss(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* d,
                                const void* observed, int kind, float grad_scale, double* loss_out, void* stream) {
    if (!s || !observed || !loss_out) return fail(LSB_EINVAL, "NULL argument");
    if ((kind & ~LSB_OBS_U8) != 0 && (kind & ~LSB_OBS_U8) != 1)
        return fail(LSB_EINVAL, "kind must be 0 (l1) or 1 (l2), optionally | LSB_OBS_U8");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    return check_cuda(launch_blend_fused(w, *s, d->width, d->height, observed, kind, grad_scale, loss_out,
                                         (cudaStream_t)stream),
                      "blend_fused_loss");
}

int lsb_render_blend_bwd_loss(const lsb_settings* s, void* ws, size_t ws_bytes, const lsb_dims* d,
                              const float* image, const void* observed, int kind, float grad_scale,
                              double* loss_out, void* stream) {
    if (!s || !observed || !loss_out) return fail(LSB_EINVAL, "NULL argument");
    if (!image) return fail(LSB_EMISSING_CACHE, "render outputs missing");
    if ((kind & ~LSB_OBS_U8) != 0 && (kind & ~LSB_OBS_U8) != 1)
        return fail(LSB_EINVAL, "kind must be 0 (l1) or 1 (l2), optionally | LSB_OBS_U8");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    return check_cuda(launch_blend_bwd_loss(w, *s, d->width, d->height, image, observed, kind, grad_scale, loss_out,
                                            (cudaStream_t)stream),
                      "blend_bwd_loss");
}

int lsb_render_chain(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s,
                     void* ws, size_t ws_bytes, const lsb_dims* d, const lsb_grads* g, double* pose_out,
                     void* stream) {
    if (!cam || !T || !s || !g) return fail(LSB_EINVAL, "NULL argument");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    rc = params_ok(p, d);
    if (rc) return rc;
    if (p->n > 0 && (!g->mean || !g->rot || !g->scale || !g->opacity || !g->sh))
        return fail(LSB_EINVAL, "NULL gradient array");
    return check_cuda(launch_chain(w, *p, *g, *cam, *T, *s, pose_out, (cudaStream_t)stream), "chain");
}

int lsb_adam_step(const lsb_params* p, const float* grads, void* m, void* v, uint8_t* touched,
                  const lsb_adam_cfg* cfg, void* stream) {
    if (!p || !cfg) return fail(LSB_EINVAL, "NULL argument");
    if (p->n > 0 && (!grads || !m || !v || !touched || !p->means || !p->rots || !p->scales || !p->opacities ||
                     !p->shs))
        return fail(LSB_EINVAL, "NULL array");
    if (cfg->step < 1) return fail(LSB_EINVAL, "Adam step count must be >= 1");
    return check_cuda(launch_adam(*p, grads, m, v, touched, *cfg, nullptr, 0, nullptr, (cudaStream_t)stream),
                      "adam");
}

int lsb_adam_step_dev(const lsb_params* p, const float* grads, void* m, void* v, uint8_t* touched,
                      const lsb_adam_cfg* cfg, const double* ibc_table, int64_t table_len, int64_t* step_dev,
                      void* stream) {
    if (!p || !cfg || !ibc_table || !step_dev) return fail(LSB_EINVAL, "NULL argument");
    if (table_len < 1) return fail(LSB_EINVAL, "empty bias-correction table");
    if (p->n > 0 && (!grads || !m || !v || !touched || !p->means || !p->rots || !p->scales || !p->opacities ||
                     !p->shs))
        return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_adam(*p, grads, m, v, touched, *cfg, ibc_table, table_len, step_dev,
                                  (cudaStream_t)stream), "adam_dev");
}

int lsb_adam_step_dev_groups(const lsb_params* p, const float* grads, void* m, void* v, uint8_t* touched,
                             const lsb_adam_cfg* cfg, const double* ibc_table, int64_t table_len,
                             int64_t* step_dev, int32_t groups, int32_t advance, void* stream) {
    if (!p || !cfg || !ibc_table || !step_dev) return fail(LSB_EINVAL, "NULL argument");
    if (table_len < 1) return fail(LSB_EINVAL, "empty bias-correction table");
    if (groups & ~LSB_ADAM_ALL) return fail(LSB_EINVAL, "unknown parameter group bits");
    if (!adam_groups_contiguous(groups)) return fail(LSB_EINVAL, "non-rotation groups must be contiguous");
    if (p->n > 0 && (!grads || !m || !v || !touched || !p->means || !p->rots || !p->scales || !p->opacities ||
                     !p->shs))
        return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_adam(*p, grads, m, v, touched, *cfg, ibc_table, table_len, step_dev,
                                  (cudaStream_t)stream, groups, advance != 0), "adam_dev_groups");
}

int lsb_copy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
    if (bytes == 0) return LSB_OK;
    if (!dst || !src) return fail(LSB_EINVAL, "NULL argument");
    return check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream), "copy_h2d");
}

int lsb_orthonormalize(void* rots, int32_t dtype, const uint8_t* touched, int64_t n, void* stream) {
    if (n > 0 && (!rots || !touched)) return fail(LSB_EINVAL, "NULL array");
    if (dtype != 0 && dtype != 1) return fail(LSB_EINVAL, "dtype must be 0 (f32) or 1 (f64)");
    return check_cuda(launch_orthonormalize(rots, dtype, touched, n, (cudaStream_t)stream), "orthonormalize");
}

int lsb_pose_prepare(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s,
                     void* ws, size_t ws_bytes, const lsb_dims* d, float* chain, void* stream) {
    if (!cam || !T || !s || !chain) return fail(LSB_EINVAL, "NULL argument");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    rc = params_ok(p, d);
    if (rc) return rc;
    return check_cuda(launch_pose_prepare(w, *p, *cam, *T, *s, chain, (cudaStream_t)stream), "pose_prepare");
}

int lsb_pose_rows(const lsb_settings* s, int sh_degree_used, void* ws, size_t ws_bytes, const lsb_dims* d,
                  const float* image, const int32_t* n_contrib, const float* chain, const int32_t* ids, int64_t m,
                  const int64_t* m_dev, const double* A, const double* R_cw, double* rows, void* stream) {
    if (!s || !A || !R_cw) return fail(LSB_EINVAL, "NULL argument");
    if (m > 0 && (!image || !n_contrib || !chain || !ids || !rows)) return fail(LSB_EINVAL, "NULL array");
    Ws w;
    int rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    return check_cuda(launch_pose_rows(w, *s, sh_degree_used, d->width, d->height, image, n_contrib, chain, ids, m,
                                       m_dev, A, R_cw, rows, (cudaStream_t)stream), "pose_rows");
}

int lsb_hb_scratch_doubles(void) { return hb_scratch_doubles(); }

int lsb_hb_reduce(const double* rows, const double* z, int64_t m, const int64_t* m_dev, double inv_sigma2,
                  double* out, double* scratch, void* stream) {
    if (!out || !scratch || (m > 0 && (!rows || !z))) return fail(LSB_EINVAL, "NULL argument");
    return check_cuda(launch_hb(rows, z, m, m_dev, inv_sigma2, out, scratch, (cudaStream_t)stream), "hb_reduce");
}

int lsb_semidense_mask(const void* obs, int32_t observed_u8, const float* tfin, int32_t W, int32_t H, double thr,
                       double tmax, uint8_t* out, void* stream) {
    if (!obs || !tfin || !out || W <= 0 || H <= 0) return fail(LSB_EINVAL, "bad argument");
    return check_cuda(launch_semidense(obs, observed_u8 != 0, tfin, W, H, thr, tmax, out, (cudaStream_t)stream),
                      "semidense");
}

static int vox_ok(const lsb_voxmap* m) {
    if (!m || !m->keys || !m->count || !m->sum || !m->outer || !m->gslot || !m->claim || !m->n_used || !m->flags)
        return fail(LSB_EINVAL, "voxmap: NULL array");
    if ((m->gkeys == nullptr) != (m->n_gkeys == nullptr))
        return fail(LSB_EINVAL, "voxmap: gkeys and n_gkeys go together");
    if (m->cap < 2 || (m->cap & (m->cap - 1))) return fail(LSB_EINVAL, "voxmap: cap must be a power of two");
    if (!(m->root_len > 0.0)) return fail(LSB_EINVAL, "root_len must be positive");
    if (m->max_level < 0 || m->max_level > 16) return fail(LSB_EINVAL, "max_level out of range");
    return LSB_OK;
}

int lsb_voxmap_keys(const double* pts, int64_t n, double edge, int64_t* out, void* stream) {
    if (n > 0 && (!pts || !out)) return fail(LSB_EINVAL, "NULL argument");
    if (!(edge > 0.0)) return fail(LSB_EINVAL, "root voxel length must be positive");
    return check_cuda(launch_vox_keys(pts, n, edge, out, (cudaStream_t)stream), "voxmap_keys");
}

int lsb_voxmap_insert_points(const lsb_voxmap* m, const double* pts, int64_t n, int32_t accumulate, int64_t* slots,
                             void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (n > 0 && !pts) return fail(LSB_EINVAL, "NULL points");
    return check_cuda(launch_vox_insert(*m, pts, n, accumulate, slots, (cudaStream_t)stream), "voxmap_insert");
}

int lsb_voxmap_accumulate_temp_bytes(int64_t n, size_t* bytes) {
    if (!bytes || n < 0) return fail(LSB_EINVAL, "bad argument");
    *bytes = vox_accumulate_temp_bytes(n);
    return LSB_OK;
}

int lsb_voxmap_accumulate(const lsb_voxmap* m, const double* pts, int64_t n, int64_t* slots, void* temp,
                          size_t temp_bytes, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (n < 0 || n > 0x7fffffffll) return fail(LSB_EINVAL, "bad n");
    if (n > 0 && (!pts || !temp)) return fail(LSB_EINVAL, "NULL argument");
    if (temp_bytes < vox_accumulate_temp_bytes(n)) return fail(LSB_EINVAL, "accumulate workspace too small");
    return check_cuda(launch_vox_accumulate(*m, pts, n, slots, temp, (cudaStream_t)stream), "voxmap_accumulate");
}

int lsb_voxmap_try_insert(const lsb_voxmap* m, const double* means, int64_t n, int32_t first_gid, int64_t* slots,
                          int32_t* status, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (n > 0 && (!means || !slots || !status)) return fail(LSB_EINVAL, "NULL argument");
    return check_cuda(launch_vox_try_insert(*m, means, n, first_gid, slots, status, (cudaStream_t)stream),
                      "voxmap_try_insert");
}

int lsb_voxmap_lookup(const lsb_voxmap* m, const int64_t* keys, int64_t n, int64_t* out, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (n > 0 && (!keys || !out)) return fail(LSB_EINVAL, "NULL argument");
    return check_cuda(launch_vox_lookup(*m, keys, n, out, (cudaStream_t)stream), "voxmap_lookup");
}

int lsb_voxmap_fov(const lsb_voxmap* m, const double* pts, int64_t n, uint64_t* rset, int64_t rcap, int64_t* out,
                   uint64_t* n_out, int64_t out_cap, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (!rset || !n_out || (out_cap > 0 && !out) || (n > 0 && !pts)) return fail(LSB_EINVAL, "NULL argument");
    if (rcap < 2 || (rcap & (rcap - 1))) return fail(LSB_EINVAL, "rcap must be a power of two");
    return check_cuda(launch_vox_fov(*m, pts, n, (unsigned long long*)rset, rcap, out, (unsigned long long*)n_out,
                                     out_cap, (cudaStream_t)stream), "voxmap_fov");
}

int lsb_voxmap_dump(const lsb_voxmap* m, int64_t* keys, int64_t* slots, uint64_t* n_out, int64_t out_cap,
                    void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (!n_out || (out_cap > 0 && (!keys || !slots))) return fail(LSB_EINVAL, "NULL argument");
    return check_cuda(launch_vox_dump(*m, keys, slots, (unsigned long long*)n_out, out_cap, (cudaStream_t)stream),
                      "voxmap_dump");
}

int lsb_voxmap_rehash(const lsb_voxmap* src, const lsb_voxmap* dst, void* stream) {
    int rc = vox_ok(src);
    if (rc) return rc;
    rc = vox_ok(dst);
    if (rc) return rc;
    return check_cuda(launch_vox_rehash(*src, *dst, (cudaStream_t)stream), "voxmap_rehash");
}

int lsb_photometric_loss(const float* rendered, const void* observed, const uint8_t* mask, int64_t npx,
                         int64_t mask_count, int kind, float grad_scale, float* grad_out,
                         double* sums_out, void* stream) {
    (void)mask_count;
    if (!rendered || !observed || !sums_out) return fail(LSB_EINVAL, "NULL argument");
    if ((kind & ~LSB_OBS_U8) != 0 && (kind & ~LSB_OBS_U8) != 1)
        return fail(LSB_EINVAL, "kind must be 0 (l1) or 1 (l2), optionally | LSB_OBS_U8");
    return check_cuda(launch_loss(rendered, observed, mask, npx, kind, grad_scale, grad_out, sums_out,
                                  (cudaStream_t)stream),
                      "loss");
}

static int arena_ok(const lsb_params* a) {
    if (!a || !a->means || !a->rots || !a->scales || !a->opacities || !a->shs) return fail(LSB_EINVAL, "NULL arena");
    if (a->dtype != 0) return fail(LSB_EINVAL, "the window arena is f32");
    if (a->sh_coeffs < 1 || a->sh_coeffs > 16) return fail(LSB_EINVAL, "sh_coeffs must be in [1, 16]");
    return LSB_OK;
}

int lsb_window_mark(const int64_t* wkeys, int64_t n, uint64_t* hkeys, int32_t* hslots, int64_t hcap,
                    const int64_t* fov, int64_t m, uint8_t* keep, uint8_t* is_add, void* stream) {
    if (n < 0 || m < 0) return fail(LSB_EINVAL, "negative count");
    if (hcap <= 0 || (hcap & (hcap - 1)) || hcap < 2 * n) return fail(LSB_EINVAL, "window hash capacity");
    if (!hkeys || !hslots || (n && (!wkeys || !keep)) || (m && (!fov || !is_add)))
        return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_win_mark(wkeys, n, hkeys, hslots, hcap, fov, m, keep, is_add, (cudaStream_t)stream),
                      "window_mark");
}

int64_t lsb_window_plan_tiles(int64_t n) { return n > 0 ? win_plan_tiles(n) : 0; }
int64_t lsb_window_append_tiles(int64_t cnt) { return cnt > 0 ? win_append_tiles(cnt) : 0; }

int lsb_window_plan(const uint8_t* keep, int64_t n, int32_t* dels, int32_t* movers, int64_t* counts, int32_t* tiles,
                    void* stream) {
    if (n < 0 || !counts || (n && (!keep || !dels || !movers || !tiles))) return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_win_plan(keep, n, dels, movers, counts, tiles, (cudaStream_t)stream), "window_plan");
}

int lsb_window_compact(const lsb_voxmap* m, const lsb_params* arena, int64_t* wkeys, const int32_t* dels, int64_t k,
                       const int32_t* movers, int64_t h, int64_t n, float* store, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    rc = arena_ok(arena);
    if (rc) return rc;
    if (k < 0 || h < 0 || h > k || k > n) return fail(LSB_EINVAL, "bad counts");
    if (k && (!dels || !store || !wkeys)) return fail(LSB_EINVAL, "NULL array");
    if (h && !movers) return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_win_compact(*m, *arena, wkeys, dels, k, movers, h, n, store, (cudaStream_t)stream),
                      "window_compact");
}

int lsb_window_leaf_gids(const lsb_voxmap* m, const int64_t* okeys, int64_t cnt, int32_t* gids, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (cnt < 0 || (cnt && (!okeys || !gids))) return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_win_leaf_gids(*m, okeys, cnt, gids, (cudaStream_t)stream), "window_leaf_gids");
}

int lsb_window_dist(const int64_t* okeys, int64_t cnt, double edge, const double* origin, double* out,
                    void* stream) {
    if (!origin || cnt < 0 || (cnt && (!okeys || !out))) return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_win_dist(okeys, cnt, edge, origin, out, (cudaStream_t)stream), "window_dist");
}

int lsb_window_append(const lsb_params* arena, int64_t* wkeys, const int64_t* okeys, const int32_t* gids, int64_t cnt,
                      const float* store, int64_t first_slot, int64_t* n_added, int32_t* tiles, void* stream) {
    int rc = arena_ok(arena);
    if (rc) return rc;
    if (!n_added || cnt < 0 || (cnt && (!okeys || !gids || !store || !wkeys || !tiles)))
        return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_win_append(*arena, wkeys, okeys, gids, cnt, store, first_slot, n_added, tiles,
                                        (cudaStream_t)stream),
                      "window_append");
}

int lsb_voxmap_fit_planes(const lsb_voxmap* m, const int64_t* keys, int64_t k, const double* origin, double* normals,
                          double* anchors, uint8_t* valid, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (!origin || k < 0 || (k && (!keys || !normals || !anchors || !valid))) return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_fit_planes(*m, keys, k, origin, normals, anchors, valid, (cudaStream_t)stream),
                      "fit_planes");
}

int lsb_lidar_rows(const lsb_voxmap* m, const double* pts_l, int64_t n, const double* R_il, const double* t_il,
                   const double* R_wi, const double* t_wi, double gate, double* rows, double* z, uint8_t* keep,
                   void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (!R_il || !t_il || !R_wi || !t_wi || n < 0 || (n && (!pts_l || !rows || !z || !keep)))
        return fail(LSB_EINVAL, "NULL array");
    const double leaf_len = m->root_len / (double)(1ll << m->max_level);
    return check_cuda(launch_lidar_rows(*m, pts_l, n, R_il, t_il, R_wi, t_wi, leaf_len, gate, rows, z, keep,
                                        (cudaStream_t)stream),
                      "lidar_rows");
}

int lsb_init_gaussians(const lsb_voxmap* m, const int64_t* keys, const double* centroids, int64_t k,
                       const float* image, int32_t width, int32_t height, const double* R_cw, const double* t_cw,
                       const double* cam4, const double* origin, double near, double kappa, double delta,
                       double opacity, int32_t sh_coeffs, float* rows, uint8_t* status, void* stream) {
    int rc = vox_ok(m);
    if (rc) return rc;
    if (!R_cw || !t_cw || !cam4 || !origin || k < 0 || (k && (!keys || !centroids || !image || !rows || !status)))
        return fail(LSB_EINVAL, "NULL array");
    if (width < 4 || height < 4 || sh_coeffs < 1 || sh_coeffs > 16) return fail(LSB_EINVAL, "bad image / sh size");
    return check_cuda(launch_init_gaussians(*m, keys, centroids, k, image, width, height, R_cw, t_cw, cam4, origin, near,
                                            kappa, delta, opacity, sh_coeffs, rows, status, (cudaStream_t)stream),
                      "init_gaussians");
}

int lsb_segment_mean(const double* pts, const int64_t* perm, const int64_t* starts, const int64_t* counts, int64_t k,
                     double* out, void* stream) {
    if (k < 0 || (k && (!pts || !perm || !starts || !counts || !out))) return fail(LSB_EINVAL, "NULL array");
    return check_cuda(launch_segment_mean(pts, perm, starts, counts, k, out, (cudaStream_t)stream), "segment_mean");
}

int lsb_adam_peer_step(const lsb_params* replicas, int32_t n_ranks, int32_t rank, const float* const* grads,
                       int64_t lo, int64_t hi, void* m, void* v, uint8_t* const* touched, const lsb_adam_cfg* cfg,
                       const double* ibc_table, int64_t table_len, int64_t* step_dev, void* stream) {
    if (!replicas || !grads || !touched || !cfg || !m || !v) return fail(LSB_EINVAL, "NULL argument");
    if (n_ranks < 1 || n_ranks > adam_max_peers() || rank < 0 || rank >= n_ranks)
        return fail(LSB_EINVAL, "rank / n_ranks out of range (at most 8 ranks)");
    const lsb_params& p = replicas[rank];
    if (lo < 0 || hi < lo || hi > p.n) return fail(LSB_EINVAL, "bad shard");
    for (int q = 0; q < n_ranks; ++q) {
        if (!grads[q] || !touched[q] || replicas[q].n != p.n || replicas[q].dtype != p.dtype ||
            replicas[q].sh_coeffs != p.sh_coeffs)
            return fail(LSB_EINVAL, "replicas / gradient buffers disagree");
    }
    if ((ibc_table != nullptr) != (step_dev != nullptr)) return fail(LSB_EINVAL, "ibc_table and step_dev go together");
    return check_cuda(launch_adam_peer(replicas, n_ranks, rank, grads, lo, hi, m, v, touched, *cfg, ibc_table,
                                       table_len, step_dev, (cudaStream_t)stream),
                      "adam_peer");
}

int64_t lsb_visual_select_scratch_bytes(int64_t npx, int32_t budget) {
    return visual_select_scratch_bytes(npx, budget);
}

int lsb_visual_select(const uint8_t* mask, const void* observed, int32_t observed_u8, const float* image, int64_t npx,
                      int32_t budget,
                      double gate, void* scratch, int32_t* ids_out, double* res_out, int64_t* counts, void* stream) {
    if (!mask || !observed || !image || !scratch || !ids_out || !res_out || !counts || npx < 0 || budget < 1)
        return fail(LSB_EINVAL, "bad argument");
    return check_cuda(launch_visual_select(mask, observed, observed_u8 != 0, image, npx, budget, gate, scratch, ids_out,
                                           res_out, counts, (cudaStream_t)stream),
                      "visual_select");
}

int lsb_visual_pass(const lsb_params* p, const lsb_camera* cam, const lsb_pose* T, const lsb_settings* s,
                    void* ws, size_t ws_bytes, const lsb_dims* d, float* image, float* t_final, int32_t* n_contrib,
                    const void* observed, const lsb_visual_cfg* c, const lsb_visual_bufs* b, void* stream) {
    if (!p || !cam || !T || !s || !c || !b || !observed) return fail(LSB_EINVAL, "NULL argument");
    if (!image || !t_final || !n_contrib || !b->mask || !b->select_scratch || !b->ids || !b->res || !b->chain ||
        !b->rows || !b->hb_scratch || !b->out || c->budget < 1)
        return fail(LSB_EINVAL, "bad buffers");
    int rc = lsb_render_fwd(p, cam, T, s, ws, ws_bytes, d, image, t_final, n_contrib, nullptr, stream);
    if (rc) return rc;
    Ws w;
    rc = get_ws(ws, ws_bytes, d, &w);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t npx = (int64_t)d->width * d->height;
    const bool u8 = c->observed_u8 != 0;
    int64_t* cnt = b->out;
    const int64_t* kept = cnt + 2;
    rc = check_cuda(launch_semidense(observed, u8, t_final, d->width, d->height, c->grad_thr, c->t_max, b->mask, st),
                    "semidense");
    if (rc) return rc;
    rc = check_cuda(launch_visual_select(b->mask, observed, u8, image, npx, c->budget, c->gate, b->select_scratch,
                                         b->ids, b->res, cnt, st),
                    "visual_select");
    if (rc) return rc;
    rc = check_cuda(launch_pose_prepare(w, *p, *cam, *T, *s, b->chain, st), "pose_prepare");
    if (rc) return rc;
    rc = check_cuda(launch_pose_rows(w, *s, c->sh_degree_used, d->width, d->height, image, n_contrib, b->chain, b->ids,
                                     c->budget, kept, c->A, T->R, b->rows, st),
                    "pose_rows");
    if (rc) return rc;
    rc = check_cuda(launch_hb(b->rows, b->res, c->budget, kept, c->inv_sigma2, (double*)(b->out + 6), b->hb_scratch, st),
                    "hb_reduce");
    if (rc) return rc;
    return check_cuda(cudaMemcpyAsync(cnt + 3, w.ctr, 3 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st), "counters");
}

int lsb_ieskf_gain(const double* cov, const double* jinv3, const double* A6, const double* b6, const double* delta,
                   double* xi, double* KH, double* P) {
    if (!cov || !jinv3 || !A6 || !b6 || !delta || !xi || !KH || !P) return fail(LSB_EINVAL, "NULL argument");
    const int r = ieskf_gain(cov, jinv3, A6, b6, delta, xi, KH, P);
    if (r == 1) return fail(LSB_EINVAL, "singular matrix");
    if (r == 2) return fail(LSB_EINVAL, "non-finite gain");
    return LSB_OK;
}

int lsb_ieskf_iterate(const double* cov, const double* x_bar, double* x_hat, const double* A6, const double* b6,
                      double bias_limit, double* xi, double* KH, double* P) {
    if (!cov || !x_bar || !x_hat || !A6 || !b6 || !xi || !KH || !P) return fail(LSB_EINVAL, "NULL argument");
    const int r = ieskf_iterate(cov, x_bar, x_hat, A6, b6, bias_limit, xi, KH, P);
    if (r == 1) return fail(LSB_EINVAL, "singular matrix");
    if (r == 2) return fail(LSB_EINVAL, "non-finite gain");
    return LSB_OK;
}

}  // extern "C"
