// K7 Adam in storage coordinates (optimize.py:103-119, 159-201), one thread
// per Gaussian, and the Gram-Schmidt re-orthonormalisation of touched
// rotations (optimize.py:91-100, 193-194).  HBM-bound: params are updated in
// place in the f32 window arena, moments are f32, arithmetic is f64.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

struct AdamArgs {
    float* means;
    float* rots;
    float* scales;
    float* opac;
    float* shs;
    int64_t n;
    int K;
    const float* g;     // flat gradient [mean 3n | rot 3n | scale 3n | opac n | sh 3Kn]
    float* m;           // flat first moments, same layout
    float* v;           // flat second moments
    uint8_t* touched;   // rotation rows stepped at least once
    lsb_adam_cfg c;
    double bc1, bc2;    // 1 - beta^t
};

__device__ __forceinline__ double adam_upd(const AdamArgs& a, int64_t idx, double g, double lr) {
    const double m = a.c.beta1 * (double)a.m[idx] + (1.0 - a.c.beta1) * g;
    const double v = a.c.beta2 * (double)a.v[idx] + (1.0 - a.c.beta2) * g * g;
    a.m[idx] = (float)m;
    a.v[idx] = (float)v;
    return -lr * (m / a.bc1) / (sqrt(v / a.bc2) + a.c.eps);
}

__global__ void __launch_bounds__(256) k_adam(AdamArgs a) {
    const int64_t n = a.n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t o_rot = 3 * n, o_scale = 6 * n, o_op = 9 * n, o_sh = 10 * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        // means
        for (int k = 0; k < 3; ++k) {
            const double st = adam_upd(a, 3 * i + k, a.g[3 * i + k], a.c.lr_mean * a.c.scene_scale);
            a.means[3 * i + k] = (float)((double)a.means[3 * i + k] + st);
        }
        // rotation: R <- R Exp(phi) on rows with phi != 0
        double phi[3];
        for (int k = 0; k < 3; ++k) phi[k] = adam_upd(a, o_rot + 3 * i + k, a.g[o_rot + 3 * i + k], a.c.lr_rot);
        if (phi[0] != 0.0 || phi[1] != 0.0 || phi[2] != 0.0) {
            const double th = sqrt(phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2]);
            const bool small = th < 1e-8;
            const double ca = small ? 1.0 : sin(th) / th;
            const double cb = small ? 0.5 : (1.0 - cos(th)) / (th * th);
            const double S[9] = {0.0, -phi[2], phi[1], phi[2], 0.0, -phi[0], -phi[1], phi[0], 0.0};
            double E[9];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    const double s2 = S[3 * r] * S[c] + S[3 * r + 1] * S[3 + c] + S[3 * r + 2] * S[6 + c];
                    E[3 * r + c] = (r == c ? 1.0 : 0.0) + ca * S[3 * r + c] + cb * s2;
                }
            float* R = a.rots + 9 * i;
            double Rd[9];
            for (int k = 0; k < 9; ++k) Rd[k] = R[k];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                    R[3 * r + c] = (float)(Rd[3 * r] * E[c] + Rd[3 * r + 1] * E[3 + c] + Rd[3 * r + 2] * E[6 + c]);
            a.touched[i] = 1;
        }
        // scale in log space; gradient chained by the current scale
        for (int k = 0; k < 3; ++k) {
            const double s = a.scales[3 * i + k];
            const double st = adam_upd(a, o_scale + 3 * i + k, (double)a.g[o_scale + 3 * i + k] * s, a.c.lr_scale);
            if (st != 0.0)
                a.scales[3 * i + k] = (float)fmax(exp(log(fmax(s, a.c.scale_floor)) + st), a.c.scale_floor);
        }
        // opacity in logit space
        {
            const double op = a.opac[i];
            const double oc = fmin(fmax(op, a.c.opacity_clip), 1.0 - a.c.opacity_clip);
            const double st = adam_upd(a, o_op + i, (double)a.g[o_op + i] * oc * (1.0 - oc), a.c.lr_opacity);
            if (st != 0.0) a.opac[i] = (float)(1.0 / (1.0 + exp(-(log(oc / (1.0 - oc)) + st))));
        }
        // SH coefficients
        const int64_t nk = 3 * (int64_t)a.K;
        for (int64_t k = 0; k < nk; ++k) {
            const int64_t idx = nk * i + k;
            const double st = adam_upd(a, o_sh + idx, a.g[o_sh + idx], a.c.lr_sh);
            a.shs[idx] = (float)((double)a.shs[idx] + st);
        }
    }
}

__global__ void __launch_bounds__(256) k_orthonormalize(float* rots, const uint8_t* touched, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (!touched[i]) continue;
        float* R = rots + 9 * i;
        double c0[3] = {R[0], R[3], R[6]}, c1[3] = {R[1], R[4], R[7]};
        const double n0 = sqrt(c0[0] * c0[0] + c0[1] * c0[1] + c0[2] * c0[2]);
        for (int k = 0; k < 3; ++k) c0[k] /= n0;
        const double d = c1[0] * c0[0] + c1[1] * c0[1] + c1[2] * c0[2];
        for (int k = 0; k < 3; ++k) c1[k] -= d * c0[k];
        const double n1 = sqrt(c1[0] * c1[0] + c1[1] * c1[1] + c1[2] * c1[2]);
        for (int k = 0; k < 3; ++k) c1[k] /= n1;
        const double c2[3] = {c0[1] * c1[2] - c0[2] * c1[1], c0[2] * c1[0] - c0[0] * c1[2],
                              c0[0] * c1[1] - c0[1] * c1[0]};
        for (int r = 0; r < 3; ++r) {
            R[3 * r] = (float)c0[r];
            R[3 * r + 1] = (float)c1[r];
            R[3 * r + 2] = (float)c2[r];
        }
    }
}

cudaError_t launch_adam(const lsb_params& p, const float* g, float* m, float* v, uint8_t* touched,
                        const lsb_adam_cfg& c, cudaStream_t st) {
    AdamArgs a{(float*)p.means, (float*)p.rots, (float*)p.scales, (float*)p.opacities, (float*)p.shs,
               p.n, p.sh_coeffs, g, m, v, touched, c, 0.0, 0.0};
    a.bc1 = 1.0 - pow(c.beta1, (double)c.step);
    a.bc2 = 1.0 - pow(c.beta2, (double)c.step);
    if (p.n == 0) return cudaSuccess;
    const int blocks = (int)((p.n + 255) / 256 < 148 * 8 ? (p.n + 255) / 256 : 148 * 8);
    k_adam<<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_orthonormalize(float* rots, const uint8_t* touched, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int blocks = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
    k_orthonormalize<<<blocks, 256, 0, st>>>(rots, touched, n);
    return cudaGetLastError();
}

}  // namespace lsb
