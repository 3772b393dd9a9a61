// K7 Adam in storage coordinates (optimize.py:103-119, 159-201), one thread
// per Gaussian, and the Gram-Schmidt re-orthonormalisation of touched
// rotations (optimize.py:91-100, 193-194).  HBM-bound: params are updated in
// place in the parameter arena's own type (f64 working copy or f32 arena).
// Compiled with --fmad=false: every operation rounds where numpy's does, and
// the single-GPU and fused peer kernels give the same bits.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

template <typename PT>
struct AdamArgs {
    PT* means;
    PT* rots;
    PT* scales;
    PT* opac;
    PT* shs;
    int64_t n;
    int K;
    const float* g;     // flat gradient [mean 3n | rot 3n | scale 3n | opac n | sh 3Kn]
    PT* m;              // flat first moments, same layout
    PT* v;              // flat second moments
    uint8_t* touched;   // rotation rows stepped at least once
    lsb_adam_cfg c;
    PT ibc1, ibc2;      // 1 / (1 - beta^t)
    const double* ibc_tab;   // device-step mode: per-step (ibc1, ibc2) rows
    int64_t ibc_len;
    const int64_t* step_dev; // steps taken so far
};

// AdamState.update (optimize.py:113-119): returns the additive step.
template <typename PT>
__device__ __forceinline__ PT adam_upd(const AdamArgs<PT>& a, PT ibc1, PT ibc2, int64_t idx, PT g, PT lr) {
    const PT m = (PT)a.c.beta1 * a.m[idx] + (PT)(1.0 - a.c.beta1) * g;
    const PT v = (PT)a.c.beta2 * a.v[idx] + (PT)(1.0 - a.c.beta2) * g * g;
    a.m[idx] = m;
    a.v[idx] = v;
    return -lr * (m * ibc1) / (sqrt(v * ibc2) + (PT)a.c.eps);
}

// Gradient sources: this rank's buffer, or the sum over every rank's buffer
// (peer pointers, added in rank order) for the fused peer step.
struct GradLocal {
    const float* g;
    __device__ __forceinline__ float operator()(int64_t idx) const { return g[idx]; }
};
constexpr int MAX_PEERS = 8;
struct GradPeers {
    const float* g[MAX_PEERS];
    int G;
    __device__ __forceinline__ float operator()(int64_t idx) const {
        float s = g[0][idx];
        for (int q = 1; q < G; ++q) s += g[q][idx];
        return s;
    }
};

// Parameter targets: read from this rank's arrays; write to them, or to
// every replica (peer pointers) so all ranks hold the same bits.
template <typename PT>
struct ParamLocal {
    PT *means, *rots, *scales, *opac, *shs;
    uint8_t* touched;
    __device__ __forceinline__ PT get(const PT* base, int64_t idx) const { return base[idx]; }
    __device__ __forceinline__ void put(int f, int64_t idx, PT v) const { field(f)[idx] = v; }
    __device__ __forceinline__ void touch(int64_t i) const { touched[i] = 1; }
    __device__ __forceinline__ PT* field(int f) const {
        return f == 0 ? means : (f == 1 ? rots : (f == 2 ? scales : (f == 3 ? opac : shs)));
    }
};
template <typename PT>
struct ParamPeers {
    PT *means, *rots, *scales, *opac, *shs;             // this rank's replica (read)
    PT* dst[MAX_PEERS][5];                               // every replica's arrays (write)
    uint8_t* touched[MAX_PEERS];
    int G;
    __device__ __forceinline__ PT* field(int f) const {
        return f == 0 ? means : (f == 1 ? rots : (f == 2 ? scales : (f == 3 ? opac : shs)));
    }
    __device__ __forceinline__ void put(int f, int64_t idx, PT v) const {
        for (int q = 0; q < G; ++q) dst[q][f][idx] = v;
    }
    __device__ __forceinline__ void touch(int64_t i) const {
        for (int q = 0; q < G; ++q) touched[q][i] = 1;
    }
};

// One Gaussian of the storage-coordinate step (optimize.py:159-188).
template <typename PT, typename GS, typename PS>
__device__ __forceinline__ void adam_gaussian(const AdamArgs<PT>& a, const GS& gs, const PS& ps, int64_t i, PT ibc1,
                                              PT ibc2) {
    const int64_t n = a.n;
    const int64_t o_rot = 3 * n, o_scale = 6 * n, o_op = 9 * n, o_sh = 10 * n;
    {
        // a row with zero gradient and zero moments (never seen by any view)
        // is an exact no-op — the reference's "a zero gradient is an exact
        // no-op" (optimize.py:164-166): skip its sqrt / division chain and
        // its stores
        const int64_t nk = 3 * (int64_t)a.K;
        bool idle = true;
        auto chk = [&](int64_t idx) { idle = idle && gs(idx) == 0.f && a.m[idx] == (PT)0 && a.v[idx] == (PT)0; };
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            chk(3 * i + k);
            chk(o_rot + 3 * i + k);
            chk(o_scale + 3 * i + k);
        }
        chk(o_op + i);
        for (int64_t k = 0; k < nk; ++k) chk(o_sh + nk * i + k);
        if (idle) return;
    }
    const PT lr_mean = (PT)(a.c.lr_mean * a.c.scene_scale), lr_rot = (PT)a.c.lr_rot;
    const PT lr_scale = (PT)a.c.lr_scale, lr_op = (PT)a.c.lr_opacity, lr_sh = (PT)a.c.lr_sh;
    const PT floor_s = (PT)a.c.scale_floor, oclip = (PT)a.c.opacity_clip;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const PT cur = ps.field(0)[3 * i + k];
        ps.put(0, 3 * i + k, cur + adam_upd(a, ibc1, ibc2, 3 * i + k, (PT)gs(3 * i + k), lr_mean));
    }
    // rotation: R <- R Exp(phi) on rows with phi != 0 (optimize.py:172-176)
    PT phi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) phi[k] = adam_upd(a, ibc1, ibc2, o_rot + 3 * i + k, (PT)gs(o_rot + 3 * i + k), lr_rot);
    if (phi[0] != (PT)0 || phi[1] != (PT)0 || phi[2] != (PT)0) {
        const double p0 = phi[0], p1 = phi[1], p2 = phi[2];
        const double th = sqrt(p0 * p0 + p1 * p1 + p2 * p2);
        const bool small = th < 1e-8;
        const double ca = small ? 1.0 : sin(th) / th;
        const double cb = small ? 0.5 : (1.0 - cos(th)) / (th * th);
        const double S[9] = {0.0, -p2, p1, p2, 0.0, -p0, -p1, p0, 0.0};
        double E[9];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double s2 = S[3 * r] * S[c] + S[3 * r + 1] * S[3 + c] + S[3 * r + 2] * S[6 + c];
                E[3 * r + c] = (r == c ? 1.0 : 0.0) + ca * S[3 * r + c] + cb * s2;
            }
        const PT* R = ps.field(1) + 9 * i;
        double Rd[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) Rd[k] = R[k];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                ps.put(1, 9 * i + 3 * r + c, (PT)(Rd[3 * r] * E[c] + Rd[3 * r + 1] * E[3 + c] + Rd[3 * r + 2] * E[6 + c]));
        ps.touch(i);
    }
    // scale in log space; gradient chained by the current scale (optimize.py:178-181)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const PT s = ps.field(2)[3 * i + k];
        const PT st = adam_upd(a, ibc1, ibc2, o_scale + 3 * i + k, (PT)gs(o_scale + 3 * i + k) * s, lr_scale);
        if (st != (PT)0) ps.put(2, 3 * i + k, fmax(exp(log(fmax(s, floor_s)) + st), floor_s));
    }
    // opacity in logit space (optimize.py:183-186)
    {
        const PT op = ps.field(3)[i];
        const PT oc = fmin(fmax(op, oclip), (PT)1 - oclip);
        const PT st = adam_upd(a, ibc1, ibc2, o_op + i, (PT)gs(o_op + i) * oc * ((PT)1 - oc), lr_op);
        if (st != (PT)0) ps.put(3, i, (PT)1 / ((PT)1 + exp(-(log(oc / ((PT)1 - oc)) + st))));
    }
    // SH coefficients
    const int64_t nk = 3 * (int64_t)a.K;
    for (int64_t k = 0; k < nk; ++k) {
        const int64_t idx = nk * i + k;
        const PT cur = ps.field(4)[idx];
        ps.put(4, idx, cur + adam_upd(a, ibc1, ibc2, o_sh + idx, (PT)gs(o_sh + idx), lr_sh));
    }
}

template <typename PT>
__device__ __forceinline__ void bias_corr(const AdamArgs<PT>& a, PT& ibc1, PT& ibc2) {
    ibc1 = a.ibc1;
    ibc2 = a.ibc2;
    if (a.ibc_tab) {
        int64_t t = *a.step_dev;
        t = t < a.ibc_len ? t : a.ibc_len - 1;
        ibc1 = (PT)a.ibc_tab[2 * t];
        ibc2 = (PT)a.ibc_tab[2 * t + 1];
    }
}

// ---- the single-GPU step as a streaming kernel ------------------------------
// The same arithmetic as adam_gaussian, element by element over the flat
// groups (mean | scale | opacity | sh: independent elements; rotation: per
// Gaussian, R <- R Exp(phi)), so the loads of four elements per thread are
// issued together and every warp access is contiguous.  An element with a
// zero gradient and zero moments is an exact no-op (its step is -0: adding
// it, or testing it against 0, changes nothing), so it is skipped without
// stores - the same bits as the per-Gaussian form.  Blocks [0, eb) take the
// elements, blocks [eb, grid) the rotations.
constexpr int ADAM_U = 4;

template <typename PT>
__device__ __forceinline__ PT adam_step_el(const lsb_adam_cfg& c, PT ibc1, PT ibc2, PT& m, PT& v, PT G, PT lr) {
    m = (PT)c.beta1 * m + (PT)(1.0 - c.beta1) * G;
    v = (PT)c.beta2 * v + (PT)(1.0 - c.beta2) * G * G;
    return -lr * (m * ibc1) / (sqrt(v * ibc2) + (PT)c.eps);
}

// The element range [ulo, uhi) of a set of non-rotation groups (contiguous
// in element order mean, scale, opacity, sh; checked by the caller).
inline void adam_group_range(int groups, int64_t n, int K, int64_t& ulo, int64_t& uhi) {
    const int64_t lo_of[4] = {0, 3 * n, 6 * n, 7 * n};
    const int64_t hi_of[4] = {3 * n, 6 * n, 7 * n, (7 + 3 * (int64_t)K) * n};
    const int bit[4] = {LSB_ADAM_MEAN, LSB_ADAM_SCALE, LSB_ADAM_OPACITY, LSB_ADAM_SH};
    ulo = uhi = 0;
    bool any = false;
    for (int q = 0; q < 4; ++q)
        if (groups & bit[q]) {
            if (!any) ulo = lo_of[q];
            uhi = hi_of[q];
            any = true;
        }
}

// True if the non-rotation groups in `groups` are contiguous in element order.
bool adam_groups_contiguous(int groups) {
    const int bit[4] = {LSB_ADAM_MEAN, LSB_ADAM_SCALE, LSB_ADAM_OPACITY, LSB_ADAM_SH};
    int first = -1, last = -1;
    for (int q = 0; q < 4; ++q)
        if (groups & bit[q]) {
            if (first < 0) first = q;
            last = q;
        }
    for (int q = first; q >= 0 && q <= last; ++q)
        if (!(groups & bit[q])) return false;
    return true;
}

// Element blocks step the elements u in [ulo, uhi) of the non-rotation
// groups — u: [0,3n) mean, [3n,6n) scale, [6n,7n) opacity, [7n, 7n + nk n)
// sh — and the blocks from `eb` on step the rotation rows (none when the
// launch has no rotation blocks).  The whole step is ulo = 0, uhi = total
// plus rotation blocks; a multi-GPU step launches one group range per
// all-reduce bucket (lsb_adam_step_dev_groups).
template <typename PT>
__global__ void __launch_bounds__(256) k_adam_flat(AdamArgs<PT> a, int eb, int64_t ulo, int64_t uhi) {
    PT ibc1, ibc2;
    bias_corr(a, ibc1, ibc2);
    const int64_t n = a.n;
    const int64_t o_rot = 3 * n, o_scale = 6 * n, o_op = 9 * n, o_sh = 10 * n;
    const PT* __restrict__ mm_ = a.m;
    const float* __restrict__ g_ = a.g;
    if ((int)blockIdx.x < eb) {
        const int64_t total = uhi;
        const int64_t stride = (int64_t)eb * blockDim.x * ADAM_U;
        for (int64_t u0 = ulo + (int64_t)blockIdx.x * blockDim.x * ADAM_U + threadIdx.x; u0 < total; u0 += stride) {
            int64_t gi[ADAM_U];
            float gr[ADAM_U];
            PT m0[ADAM_U], v0[ADAM_U], p0[ADAM_U];
            PT* pp[ADAM_U];
#pragma unroll
            for (int q = 0; q < ADAM_U; ++q) {
                const int64_t u = u0 + (int64_t)q * blockDim.x;
                int64_t j = u;
                PT* base = a.means;
                gi[q] = -1;
                if (u >= total) {
                    // past this launch's group range (another part's elements)
                } else if (u < 3 * n) {
                    gi[q] = u;
                } else if (u < 6 * n) {
                    j = u - 3 * n;
                    base = a.scales;
                    gi[q] = o_scale + j;
                } else if (u < 7 * n) {
                    j = u - 6 * n;
                    base = a.opac;
                    gi[q] = o_op + j;
                } else if (u < total) {
                    j = u - 7 * n;
                    base = a.shs;
                    gi[q] = o_sh + j;
                }
                pp[q] = base + j;
                if (gi[q] >= 0) {
                    gr[q] = g_[gi[q]];
                    m0[q] = mm_[gi[q]];
                    v0[q] = a.v[gi[q]];
                    p0[q] = *pp[q];
                }
            }
#pragma unroll
            for (int q = 0; q < ADAM_U; ++q) {
                if (gi[q] < 0) continue;
                if (gr[q] == 0.f && m0[q] == (PT)0 && v0[q] == (PT)0) continue;      // exact no-op
                const int64_t u = u0 + (int64_t)q * blockDim.x;
                PT mq = m0[q], vq = v0[q];
                if (u < 3 * n) {
                    const PT st = adam_step_el(a.c, ibc1, ibc2, mq, vq, (PT)gr[q], (PT)(a.c.lr_mean * a.c.scene_scale));
                    *pp[q] = p0[q] + st;
                } else if (u < 6 * n) {
                    const PT s = p0[q];
                    const PT st = adam_step_el(a.c, ibc1, ibc2, mq, vq, (PT)gr[q] * s, (PT)a.c.lr_scale);
                    const PT fl = (PT)a.c.scale_floor;
                    if (st != (PT)0) *pp[q] = fmax(exp(log(fmax(s, fl)) + st), fl);
                } else if (u < 7 * n) {
                    const PT oclip = (PT)a.c.opacity_clip;
                    const PT oc = fmin(fmax(p0[q], oclip), (PT)1 - oclip);
                    const PT st = adam_step_el(a.c, ibc1, ibc2, mq, vq, (PT)gr[q] * oc * ((PT)1 - oc),
                                               (PT)a.c.lr_opacity);
                    if (st != (PT)0) *pp[q] = (PT)1 / ((PT)1 + exp(-(log(oc / ((PT)1 - oc)) + st)));
                } else {
                    const PT st = adam_step_el(a.c, ibc1, ibc2, mq, vq, (PT)gr[q], (PT)a.c.lr_sh);
                    *pp[q] = p0[q] + st;
                }
                a.m[gi[q]] = mq;
                a.v[gi[q]] = vq;
            }
        }
        return;
    }
    // rotations: R <- R Exp(phi) on rows with phi != 0 (optimize.py:172-176)
    const int64_t rstride = (int64_t)(gridDim.x - eb) * blockDim.x;
    for (int64_t i = (int64_t)(blockIdx.x - eb) * blockDim.x + threadIdx.x; i < n; i += rstride) {
        float gr[3];
        PT m0[3], v0[3];
        bool idle = true;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            gr[k] = g_[o_rot + 3 * i + k];
            m0[k] = mm_[o_rot + 3 * i + k];
            v0[k] = a.v[o_rot + 3 * i + k];
            idle = idle && gr[k] == 0.f && m0[k] == (PT)0 && v0[k] == (PT)0;
        }
        if (idle) continue;
        PT phi[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            phi[k] = adam_step_el(a.c, ibc1, ibc2, m0[k], v0[k], (PT)gr[k], (PT)a.c.lr_rot);
            a.m[o_rot + 3 * i + k] = m0[k];
            a.v[o_rot + 3 * i + k] = v0[k];
        }
        if (phi[0] != (PT)0 || phi[1] != (PT)0 || phi[2] != (PT)0) {
            const double p0 = phi[0], p1 = phi[1], p2 = phi[2];
            const double th = sqrt(p0 * p0 + p1 * p1 + p2 * p2);
            const bool small = th < 1e-8;
            const double ca = small ? 1.0 : sin(th) / th;
            const double cb = small ? 0.5 : (1.0 - cos(th)) / (th * th);
            const double S[9] = {0.0, -p2, p1, p2, 0.0, -p0, -p1, p0, 0.0};
            double E[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double s2 = S[3 * r] * S[c] + S[3 * r + 1] * S[3 + c] + S[3 * r + 2] * S[6 + c];
                    E[3 * r + c] = (r == c ? 1.0 : 0.0) + ca * S[3 * r + c] + cb * s2;
                }
            PT* R = a.rots + 9 * i;
            double Rd[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) Rd[k] = R[k];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    R[3 * r + c] = (PT)(Rd[3 * r] * E[c] + Rd[3 * r + 1] * E[3 + c] + Rd[3 * r + 2] * E[6 + c]);
            a.touched[i] = 1;
        }
    }
}

// Fused multi-GPU step over NVLink peer memory (one kernel per rank): for the
// Gaussians [lo, hi) this rank owns, sum the G ranks' gradient buffers (peer
// loads, rank order — the all-reduce), apply Adam with this rank's moments,
// and store the new parameters into every rank's replica (peer stores — the
// all-gather).  Every replica receives the same bits.  The caller brackets
// it with a cross-rank barrier (gradients complete before; stores landed
// after).
template <typename PT>
__global__ void __launch_bounds__(256) k_adam_peer(AdamArgs<PT> a, GradPeers gs, ParamPeers<PT> ps, int64_t lo,
                                                   int64_t hi) {
    PT ibc1, ibc2;
    bias_corr(a, ibc1, ibc2);
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x)
        adam_gaussian(a, gs, ps, i, ibc1, ibc2);
    __threadfence_system();
}

template <typename PT>
__global__ void __launch_bounds__(256) k_orthonormalize(PT* rots, const uint8_t* touched, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (!touched[i]) continue;
        PT* R = rots + 9 * i;
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
            R[3 * r] = (PT)c0[r];
            R[3 * r + 1] = (PT)c1[r];
            R[3 * r + 2] = (PT)c2[r];
        }
    }
}

static int grid_of(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (int)(b < 148 * 8 ? b : 148 * 8);
}

__global__ void k_step_bump(int64_t* step_dev) { *step_dev += 1; }

template <typename PT>
static cudaError_t adam_t(const lsb_params& p, const float* g, void* m, void* v, uint8_t* touched,
                          const lsb_adam_cfg& c, const double* tab, int64_t tab_len, int64_t* step_dev,
                          cudaStream_t st, int groups = LSB_ADAM_ALL, bool advance = true) {
    AdamArgs<PT> a{(PT*)p.means, (PT*)p.rots, (PT*)p.scales, (PT*)p.opacities, (PT*)p.shs, p.n, p.sh_coeffs,
                   g, (PT*)m, (PT*)v, touched, c, (PT)0, (PT)0, tab, tab_len, step_dev};
    if (!tab) {
        a.ibc1 = (PT)(1.0 / (1.0 - pow(c.beta1, (double)c.step)));
        a.ibc2 = (PT)(1.0 / (1.0 - pow(c.beta2, (double)c.step)));
    }
    if (p.n > 0) {
        // element blocks (~ADAM_U elements per thread, one wave of 148 x 8 CTAs at most) + rotation blocks
        int64_t ulo = 0, uhi = 0;
        adam_group_range(groups, p.n, p.sh_coeffs, ulo, uhi);
        int64_t eb = (uhi - ulo + 256 * ADAM_U - 1) / (256 * ADAM_U);
        eb = eb < 148 * 6 ? eb : 148 * 6;
        int64_t rb = (groups & LSB_ADAM_ROT) ? (p.n + 255) / 256 : 0;
        rb = rb < 148 * 2 ? rb : 148 * 2;
        if (eb + rb > 0) k_adam_flat<PT><<<(unsigned)(eb + rb), 256, 0, st>>>(a, (int)eb, ulo, uhi);
    }
    if (step_dev && advance) k_step_bump<<<1, 1, 0, st>>>(step_dev);
    return cudaGetLastError();
}

cudaError_t launch_adam(const lsb_params& p, const float* g, void* m, void* v, uint8_t* touched,
                        const lsb_adam_cfg& c, const double* tab, int64_t tab_len, int64_t* step_dev,
                        cudaStream_t st, int groups, bool advance) {
    if (p.n == 0 && !(step_dev && advance)) return cudaSuccess;
    return p.dtype ? adam_t<double>(p, g, m, v, touched, c, tab, tab_len, step_dev, st, groups, advance)
                   : adam_t<float>(p, g, m, v, touched, c, tab, tab_len, step_dev, st, groups, advance);
}

template <typename PT>
static cudaError_t adam_peer_t(const lsb_params* reps, int G, int rank, const float* const* grads, int64_t lo,
                               int64_t hi, void* m, void* v, uint8_t* const* touched, const lsb_adam_cfg& c,
                               const double* tab, int64_t tab_len, int64_t* step_dev, cudaStream_t st) {
    const lsb_params& p = reps[rank];
    AdamArgs<PT> a{(PT*)p.means, (PT*)p.rots, (PT*)p.scales, (PT*)p.opacities, (PT*)p.shs, p.n, p.sh_coeffs,
                   nullptr, (PT*)m, (PT*)v, touched[rank], c, (PT)0, (PT)0, tab, tab_len, step_dev};
    if (!tab) {
        a.ibc1 = (PT)(1.0 / (1.0 - pow(c.beta1, (double)c.step)));
        a.ibc2 = (PT)(1.0 / (1.0 - pow(c.beta2, (double)c.step)));
    }
    GradPeers gs{};
    ParamPeers<PT> ps{};
    gs.G = ps.G = G;
    ps.means = (PT*)p.means;
    ps.rots = (PT*)p.rots;
    ps.scales = (PT*)p.scales;
    ps.opac = (PT*)p.opacities;
    ps.shs = (PT*)p.shs;
    for (int q = 0; q < G; ++q) {
        gs.g[q] = grads[q];
        ps.dst[q][0] = (PT*)reps[q].means;
        ps.dst[q][1] = (PT*)reps[q].rots;
        ps.dst[q][2] = (PT*)reps[q].scales;
        ps.dst[q][3] = (PT*)reps[q].opacities;
        ps.dst[q][4] = (PT*)reps[q].shs;
        ps.touched[q] = touched[q];
    }
    if (hi > lo) k_adam_peer<PT><<<grid_of(hi - lo), 256, 0, st>>>(a, gs, ps, lo, hi);
    if (step_dev) k_step_bump<<<1, 1, 0, st>>>(step_dev);
    return cudaGetLastError();
}

int adam_max_peers() { return MAX_PEERS; }

cudaError_t launch_adam_peer(const lsb_params* reps, int G, int rank, const float* const* grads, int64_t lo,
                             int64_t hi, void* m, void* v, uint8_t* const* touched, const lsb_adam_cfg& c,
                             const double* tab, int64_t tab_len, int64_t* step_dev, cudaStream_t st) {
    return reps[rank].dtype ? adam_peer_t<double>(reps, G, rank, grads, lo, hi, m, v, touched, c, tab, tab_len, step_dev, st)
                            : adam_peer_t<float>(reps, G, rank, grads, lo, hi, m, v, touched, c, tab, tab_len, step_dev, st);
}

cudaError_t launch_orthonormalize(void* rots, int dtype, const uint8_t* touched, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (dtype)
        k_orthonormalize<double><<<grid_of(n), 256, 0, st>>>((double*)rots, touched, n);
    else
        k_orthonormalize<float><<<grid_of(n), 256, 0, st>>>((float*)rots, touched, n);
    return cudaGetLastError();
}

}  // namespace lsb
