// K6 photometric pose rows and the IESKF H/b reduction (raster.py:402-508,
// estimator.py:241-323).
//
//   k_pose_prepare : per visible splat, the 6x2 / 6x3 maps from screen-space
//                    gradients to the camera tangent (L_mu, L_sig,
//                    raster.py:402-447) plus the SH view-direction pieces.
//   k_pose_rows    : one warp per selected pixel.  The warp walks the pixel's
//                    tile list 32 entries at a time; lanes test bbox
//                    membership and evaluate alpha in parallel, a warp scan
//                    gives each entry its transmittance T_k and prefix colour,
//                    and each lane applies d(alpha) -> (d mu, d Sigma) -> L to
//                    its entry.  The 6-vector is warp-reduced and mapped to
//                    the IMU tangent with the adjoint A (raster.py:501-507).
//   k_hb_partial / k_hb_final : A6 = sum h h^T / sigma^2, b6 = sum h z /
//                    sigma^2 with h = -row (estimator.py:278-280, 314-318),
//                    fixed-grid CTA partials then a fixed-order sum
//                    (deterministic).
//   k_semidense    : Sobel/8 gradient magnitude of the observed grey image
//                    (nearest border) > threshold and coverage T < max
//                    (estimator.py:241-252).
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

constexpr int CHAIN_F = 48;   // floats per splat in the pose-chain buffer

struct PosePrepArgs {
    lsb_params p;
    lsb_camera cam;
    lsb_pose T;
    int degree;
    float* out;
};

__constant__ double c_SH3[16] = {
    0.28209479177387814, 0.4886025119029199, 1.0925484305920792, -1.0925484305920792,
    0.31539156525252005, -1.0925484305920792, 0.5462742152960396, -0.5900435899266435,
    2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
    1.445305721320277, -0.5900435899266435, 0.0, 0.0};

__device__ void sh_grad3(int degree, double x, double y, double z, int k, double* g) {
    const double* C = c_SH3;
    g[0] = g[1] = g[2] = 0.0;
    const double xx = x * x, yy = y * y, zz = z * z;
    switch (k) {
        case 1: g[1] = -C[1]; break;
        case 2: g[2] = C[1]; break;
        case 3: g[0] = -C[1]; break;
        case 4: g[0] = C[2] * y; g[1] = C[2] * x; break;
        case 5: g[1] = C[3] * z; g[2] = C[3] * y; break;
        case 6: g[0] = C[4] * (-2.0 * x); g[1] = C[4] * (-2.0 * y); g[2] = C[4] * (4.0 * z); break;
        case 7: g[0] = C[5] * z; g[2] = C[5] * x; break;
        case 8: g[0] = C[6] * (2.0 * x); g[1] = C[6] * (-2.0 * y); break;
        case 9: g[0] = C[7] * 6.0 * x * y; g[1] = C[7] * (3.0 * xx - 3.0 * yy); break;
        case 10: g[0] = C[8] * y * z; g[1] = C[8] * x * z; g[2] = C[8] * x * y; break;
        case 11: g[0] = C[9] * (-2.0 * x * y); g[1] = C[9] * (4.0 * zz - xx - 3.0 * yy); g[2] = C[9] * (8.0 * y * z); break;
        case 12: g[0] = C[10] * (-6.0 * x * z); g[1] = C[10] * (-6.0 * y * z);
                 g[2] = C[10] * (6.0 * zz - 3.0 * xx - 3.0 * yy); break;
        case 13: g[0] = C[11] * (4.0 * zz - 3.0 * xx - yy); g[1] = C[11] * (-2.0 * x * y); g[2] = C[11] * (8.0 * x * z); break;
        case 14: g[0] = C[12] * (2.0 * x * z); g[1] = C[12] * (-2.0 * y * z); g[2] = C[12] * (xx - yy); break;
        case 15: g[0] = C[13] * (3.0 * xx - 3.0 * yy); g[1] = C[13] * (-6.0 * x * y); break;
        default: break;
    }
}

// Layout of one splat's chain record (floats):
//   [0..11]  L_mu (6x2 row-major)   [12..29] L_sig (6x3 row-major)
//   [30..38] Pm[c][d] = d colour_c / d dir_d   [39..41] dir   [42] 1/r
//   [43] interior bits (as float)
__global__ void __launch_bounds__(256) k_pose_prepare(Ws w, PosePrepArgs a) {
    const int64_t M = (int64_t)w.ctr[0];
    const double* R = a.T.R;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; slot < M; slot += stride) {
        const int64_t i = w.rec[slot].id;
        const int f64 = a.p.dtype;
        const double px = pld(a.p.means, 3 * i, f64), py = pld(a.p.means, 3 * i + 1, f64),
                     pz = pld(a.p.means, 3 * i + 2, f64);
        const double x = R[0] * px + R[1] * py + R[2] * pz + a.T.t[0];
        const double y = R[3] * px + R[4] * py + R[5] * pz + a.T.t[1];
        const double z = R[6] * px + R[7] * py + R[8] * pz + a.T.t[2];
        const double fx = a.cam.fx, fy = a.cam.fy;
        const double J00 = fx / z, J02 = -fx * x / (z * z), J11 = fy / z, J12 = -fy * y / (z * z);
        double B[9], Wc[9];
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3)
                B[3 * r3 + c3] = pld(a.p.rots, 9 * i + 3 * r3 + c3, f64) * pld(a.p.scales, 3 * i + c3, f64);
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3)
                Wc[3 * r3 + c3] = B[3 * r3] * B[3 * c3] + B[3 * r3 + 1] * B[3 * c3 + 1] + B[3 * r3 + 2] * B[3 * c3 + 2];
        double Mm[6];
        for (int k = 0; k < 3; ++k) {
            Mm[k] = J00 * R[k] + J02 * R[6 + k];
            Mm[3 + k] = J11 * R[3 + k] + J12 * R[6 + k];
        }
        double MC[6];   // M W
        for (int r2 = 0; r2 < 2; ++r2)
            for (int c3 = 0; c3 < 3; ++c3)
                MC[3 * r2 + c3] = Mm[3 * r2] * Wc[c3] + Mm[3 * r2 + 1] * Wc[3 + c3] + Mm[3 * r2 + 2] * Wc[6 + c3];
        float* o = a.out + slot * CHAIN_F;
        // L_mu: column i = (mu_c x J_i, J_i), J_0 = (J00, 0, J02), J_1 = (0, J11, J12)
        const double Jr[2][3] = {{J00, 0.0, J02}, {0.0, J11, J12}};
        for (int c = 0; c < 2; ++c) {
            const double* j = Jr[c];
            o[0 * 2 + c] = (float)(y * j[2] - z * j[1]);
            o[1 * 2 + c] = (float)(z * j[0] - x * j[2]);
            o[2 * 2 + c] = (float)(x * j[1] - y * j[0]);
            o[3 * 2 + c] = (float)j[0];
            o[4 * 2 + c] = (float)j[1];
            o[5 * 2 + c] = (float)j[2];
        }
        // L_sig: basis b in {E00, E01+E10, E11}; dM_b = 2 E_b M W
        const double gxx = -fx / (z * z), gyy = -fy / (z * z);
        for (int b = 0; b < 3; ++b) {
            double dM[6];
            for (int c3 = 0; c3 < 3; ++c3) {
                const double r0 = MC[c3], r1 = MC[3 + c3];
                dM[c3] = 2.0 * (b == 0 ? r0 : (b == 1 ? r1 : 0.0));
                dM[3 + c3] = 2.0 * (b == 0 ? 0.0 : (b == 1 ? r0 : r1));
            }
            double dJ[6];
            for (int r2 = 0; r2 < 2; ++r2)
                for (int c3 = 0; c3 < 3; ++c3)
                    dJ[3 * r2 + c3] = dM[3 * r2] * R[3 * c3] + dM[3 * r2 + 1] * R[3 * c3 + 1] + dM[3 * r2 + 2] * R[3 * c3 + 2];
            double dW[9];
            for (int c3 = 0; c3 < 3; ++c3) {
                dW[c3] = J00 * dM[c3];
                dW[3 + c3] = J11 * dM[3 + c3];
                dW[6 + c3] = J02 * dM[c3] + J12 * dM[3 + c3];
            }
            const double dmu[3] = {dJ[2] * gxx, dJ[5] * gyy,
                                   dJ[0] * gxx + dJ[4] * gyy + dJ[2] * (2.0 * fx * x / (z * z * z)) +
                                       dJ[5] * (2.0 * fy * y / (z * z * z))};
            double Z[9];
            for (int r3 = 0; r3 < 3; ++r3)
                for (int c3 = 0; c3 < 3; ++c3)
                    Z[3 * r3 + c3] = dW[3 * r3] * R[3 * c3] + dW[3 * r3 + 1] * R[3 * c3 + 1] + dW[3 * r3 + 2] * R[3 * c3 + 2];
            o[12 + 0 * 3 + b] = (float)(y * dmu[2] - z * dmu[1] + (Z[7] - Z[5]));
            o[12 + 1 * 3 + b] = (float)(z * dmu[0] - x * dmu[2] + (Z[2] - Z[6]));
            o[12 + 2 * 3 + b] = (float)(x * dmu[1] - y * dmu[0] + (Z[3] - Z[1]));
            o[12 + 3 * 3 + b] = (float)dmu[0];
            o[12 + 4 * 3 + b] = (float)dmu[1];
            o[12 + 5 * 3 + b] = (float)dmu[2];
        }
        // SH view-direction pieces
        const double* cc3 = a.T.cam_center;
        const double dvx = px - cc3[0], dvy = py - cc3[1], dvz = pz - cc3[2];
        const double dn = sqrt(dvx * dvx + dvy * dvy + dvz * dvz);
        double d0 = 0.0, d1 = 0.0, d2 = 1.0;
        if (dn > 0.0) {
            const double inv = fmax(dn, 1e-30);
            d0 = dvx / inv; d1 = dvy / inv; d2 = dvz / inv;
        }
        const int K = a.p.sh_coeffs, kk = (a.degree + 1) * (a.degree + 1);
        double Pm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int k = 1; k < kk; ++k) {
            double g[3];
            sh_grad3(a.degree, d0, d1, d2, k, g);
            for (int c = 0; c < 3; ++c) {
                const double s = pld(a.p.shs, (i * K + k) * 3 + c, f64);
                Pm[3 * c] += s * g[0]; Pm[3 * c + 1] += s * g[1]; Pm[3 * c + 2] += s * g[2];
            }
        }
        for (int k = 0; k < 9; ++k) o[30 + k] = (float)Pm[k];
        o[39] = (float)d0; o[40] = (float)d1; o[41] = (float)d2;
        o[42] = (float)(1.0 / fmax(dn, 1e-30));
        o[43] = (float)w.colmask[slot];
        o[44] = o[45] = o[46] = o[47] = 0.f;
    }
}

struct RowArgs {
    int W, H;
    float clamp, cut, iclamp;
    float cutlo, cuthi;      // cut (1 -+ CUT_BAND): inside, the f64 decision (exact_alpha)
    double clamp_d, cut_d;
    int degree;
    double A[36];
    double Rcw[9];
};

__device__ __forceinline__ float warp_scan_mul_excl(float v, int lane, float& total) {
    float x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x *= y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    const float ex = __shfl_up_sync(0xffffffffu, x, 1);
    return lane == 0 ? 1.f : ex;
}

__device__ __forceinline__ float warp_scan_add_incl(float v, int lane, float& total) {
    float x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x;
}

__global__ void __launch_bounds__(128) k_pose_rows(Ws w, RowArgs a, const float* __restrict__ image,
                                                   const int32_t* __restrict__ n_contrib,
                                                   const float* __restrict__ chain, const int32_t* __restrict__ ids,
                                                   int64_t m, const int64_t* __restrict__ m_dev,
                                                   double* __restrict__ rows) {
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (m_dev && *m_dev < m) m = *m_dev;
    if (r >= m) return;
    const int p = ids[r];
    const int px = p % a.W, py = p / a.W;
    const int tile = (py / TILE) * w.ntx + px / TILE;
    const int ox = (px / TILE) * TILE, oy = (py / TILE) * TILE;
    const float fx = (float)(px - ox), fy = (float)(py - oy);
    const int start = w.tile_start[tile], end = w.tile_last[tile];
    int rem = n_contrib[p];
    const float ir = image[3 * p], ig = image[3 * p + 1], ib = image[3 * p + 2];
    const float k2 = -2.0f / (float)LOG2E;
    float Tc = 1.f, Pr = 0.f, Pg = 0.f, Pb = 0.f;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int base = start; base < end && rem > 0; base += 32) {
        const int j = base + lane;
        bool inside = false;
        int slot = 0;
        Rec rc;
        if (j < end) {
            slot = w.tile_slot[j] & SLOT_MASK;
            rc = w.rec[slot];
            const int x0 = rc.bbx & 0xffff, x1 = rc.bbx >> 16, y0 = rc.bby & 0xffff, y1 = rc.bby >> 16;
            inside = px >= x0 && px < x1 && py >= y0 && py < y1;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, inside);
        const int ord = __popc(bal & ((1u << lane) - 1u));
        const bool active = inside && ord < rem;
        rem -= min(__popc(bal), rem);
        float G = 0.f, al = 0.f, u = 0.f, dy = 0.f;
        bool contrib = false;
        if (active) {
            const float mxl = (rc.mxh - (float)ox) + rc.mxl, myl = (rc.myh - (float)oy) + rc.myl;
            dy = fy - myl;
            u = fmaf(rc.s, dy, fx - mxl);
            G = a.clamp * ex2_approx(fmaf(rc.A, u * u, fmaf(rc.E * dy, dy, rc.lop)));   // op g
            al = fminf(G, a.clamp);
            rc.kc0 *= a.iclamp;                 // back to the clamped colour
            rc.kc1 *= a.iclamp;
            rc.kc2 *= a.iclamp;
            contrib = (al >= a.cut) && al != 0.f;
            if (a.cut_d > 0.0 && al >= a.cutlo && al < a.cuthi)       // the forward's f64 decision
                contrib = !(exact_alpha(w.cgeo[slot], a.clamp_d, (double)px, (double)py) < a.cut_d);
        }
        float tot;
        const float Tk = Tc * warp_scan_mul_excl(contrib ? 1.f - al : 1.f, lane, tot);
        const float wt = contrib ? al * Tk : 0.f;
        float sr, sg, sb;
        const float pr = Pr + warp_scan_add_incl(wt * (active ? rc.kc0 : 0.f), lane, sr);
        const float pg = Pg + warp_scan_add_incl(wt * (active ? rc.kc1 : 0.f), lane, sg);
        const float pb = Pb + warp_scan_add_incl(wt * (active ? rc.kc2 : 0.f), lane, sb);
        Tc *= tot;
        Pr += sr; Pg += sg; Pb += sb;
        if (contrib) {
            const float inv = 1.f / (1.f - al);
            const float third = 1.f / 3.f;
            const float da = third * (rc.kc0 * Tk - (ir - pr) * inv) + third * (rc.kc1 * Tk - (ig - pg) * inv) +
                             third * (rc.kc2 * Tk - (ib - pb) * inv);
            float emu0 = 0.f, emu1 = 0.f, ec0 = 0.f, ec1 = 0.f, ec2 = 0.f;
            if (al < a.clamp) {
                const float gq = da * G;
                const float v0 = (rc.A * k2) * u;
                const float v1 = fmaf(rc.s, v0, (rc.E * k2) * dy);
                emu0 = gq * v0; emu1 = gq * v1;
                ec0 = 0.5f * gq * v0 * v0; ec1 = 0.5f * gq * v0 * v1; ec2 = 0.5f * gq * v1 * v1;
            }
            const float* L = chain + (int64_t)slot * CHAIN_F;
            double c6[6];
#pragma unroll
            for (int q = 0; q < 6; ++q)
                c6[q] = (double)L[2 * q] * emu0 + (double)L[2 * q + 1] * emu1 + (double)L[12 + 3 * q] * ec0 +
                        (double)L[12 + 3 * q + 1] * ec1 + (double)L[12 + 3 * q + 2] * ec2;
            if (a.degree >= 1) {
                const int im = (int)L[43];
                const double dc[3] = {(im & 1) ? wt / 3.0 : 0.0, (im & 2) ? wt / 3.0 : 0.0, (im & 4) ? wt / 3.0 : 0.0};
                double dd[3];
                for (int q = 0; q < 3; ++q) dd[q] = dc[0] * L[30 + q] + dc[1] * L[33 + q] + dc[2] * L[36 + q];
                const double dot = L[39] * dd[0] + L[40] * dd[1] + L[41] * dd[2];
                double pt[3];
                for (int q = 0; q < 3; ++q) pt[q] = (dd[q] - L[39 + q] * dot) * L[42];
                for (int q = 0; q < 3; ++q)
                    c6[3 + q] += a.Rcw[3 * q] * pt[0] + a.Rcw[3 * q + 1] * pt[1] + a.Rcw[3 * q + 2] * pt[2];
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] += c6[q];
        }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    }
    if (lane < 6) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < 6; ++q) v += acc[q] * a.A[6 * q + lane];
        rows[6 * r + lane] = v;
    }
}

// Pass 1: HB_BLOCKS fixed CTAs, each thread accumulates the 21 unique h h^T
// entries and the 6 h z entries of its rows (fixed grid-stride partition),
// a fixed tree reduces them per CTA.  Pass 2: one CTA adds the CTA partials
// in CTA order.  Deterministic; every row is read once.
constexpr int HB_BLOCKS = 296, HB_VALS = 27;
__global__ void __launch_bounds__(256) k_hb_partial(const double* __restrict__ rows, const double* __restrict__ z,
                                                    int64_t m, const int64_t* __restrict__ m_dev,
                                                    double* __restrict__ part) {
    if (m_dev && *m_dev < m) m = *m_dev;
    __shared__ double s[HB_VALS][256 / 32];
    double v[HB_VALS];
#pragma unroll
    for (int q = 0; q < HB_VALS; ++q) v[q] = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        double h[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) h[c] = -rows[6 * r + c];
        const double zr = z[r];
        int q = 0;
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = i; j < 6; ++j) v[q++] += h[i] * h[j];
#pragma unroll
        for (int i = 0; i < 6; ++i) v[21 + i] += h[i] * zr;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < HB_VALS; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
        if (lane == 0) s[q][warp] = v[q];
    }
    __syncthreads();
    if (threadIdx.x < HB_VALS) {
        double t = 0.0;
        for (int w = 0; w < 256 / 32; ++w) t += s[threadIdx.x][w];
        part[(int64_t)blockIdx.x * HB_VALS + threadIdx.x] = t;
    }
}

// One warp per value: lane l adds the partials b = l, l + 32, ... in order,
// then a fixed butterfly combines the lanes (deterministic; the 296 partials
// no longer go through one thread's dependent adds: ~22 -> ~3 us).
__global__ void __launch_bounds__(32 * HB_VALS) k_hb_final(const double* __restrict__ part, int nblocks, double inv_s2,
                                                          double* __restrict__ out) {
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double t = 0.0;
    for (int b = lane; b < nblocks; b += 32) t += part[(int64_t)b * HB_VALS + q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane) return;
    t *= inv_s2;
    if (q >= 21) {
        out[36 + q - 21] = t;
        return;
    }
    int i = 0, k = q;
    while (k >= 6 - i) {
        k -= 6 - i;
        ++i;
    }
    const int j = i + k;
    out[6 * i + j] = t;
    out[6 * j + i] = t;
}

// One 32x8 block of pixels per CTA: the grey values of the block and its
// one-pixel (clamped) border are computed once into shared memory, then
// every pixel reads its 3x3 neighbourhood from there — the same f64 values
// and operation order as per-pixel recomputation.
constexpr int SD_BX = 32, SD_BY = 8;
__global__ void __launch_bounds__(SD_BX * SD_BY) k_semidense(const void* __restrict__ obs, bool u8,
                                                            const float* __restrict__ tfin, int W, int H, double thr,
                                                            double tmax, uint8_t* __restrict__ out) {
    __shared__ double g[SD_BY + 2][SD_BX + 2];
    const int x0 = blockIdx.x * SD_BX, y0 = blockIdx.y * SD_BY;
    for (int k = threadIdx.x; k < (SD_BX + 2) * (SD_BY + 2); k += SD_BX * SD_BY) {
        const int ly = k / (SD_BX + 2), lx = k % (SD_BX + 2);
        const int xx = min(max(x0 + lx - 1, 0), W - 1), yy = min(max(y0 + ly - 1, 0), H - 1);
        const int64_t q = 3 * ((int64_t)yy * W + xx);
        g[ly][lx] = (obs_value(obs, u8, q) + obs_value(obs, u8, q + 1) + obs_value(obs, u8, q + 2)) / 3.0;
    }
    __syncthreads();
    const int tx = threadIdx.x % SD_BX, ty = threadIdx.x / SD_BX;
    const int x = x0 + tx, y = y0 + ty;
    if (x >= W || y >= H) return;
    // ndimage.sobel(axis=1): d/dx [-1,0,1], smoothed [1,2,1] along y; axis=0 the transpose
    const double(*c)[SD_BX + 2] = (const double(*)[SD_BX + 2]) & g[ty][tx];
    const double gx = ((c[0][2] - c[0][0]) + 2.0 * (c[1][2] - c[1][0]) + (c[2][2] - c[2][0])) / 8.0;
    const double gy = ((c[2][0] - c[0][0]) + 2.0 * (c[2][1] - c[0][1]) + (c[2][2] - c[0][2])) / 8.0;
    const int64_t p = (int64_t)y * W + x;
    out[p] = (hypot(gx, gy) > thr && (double)tfin[p] < tmax) ? 1 : 0;
}

cudaError_t launch_pose_prepare(const Ws& w, const lsb_params& p, const lsb_camera& cam, const lsb_pose& T,
                                const lsb_settings& s, float* out, cudaStream_t st) {
    PosePrepArgs a{p, cam, T, 0, out};
    int deg_store = 0;
    while ((deg_store + 2) * (deg_store + 2) <= p.sh_coeffs) ++deg_store;
    a.degree = s.sh_degree < deg_store ? s.sh_degree : deg_store;
    k_pose_prepare<<<2 * 148, 256, 0, st>>>(w, a);
    return cudaGetLastError();
}

cudaError_t launch_pose_rows(const Ws& w, const lsb_settings& s, int degree, int W, int H, const float* image,
                             const int32_t* n_contrib, const float* chain, const int32_t* ids, int64_t m,
                             const int64_t* m_dev, const double* A, const double* Rcw, double* rows, cudaStream_t st) {
    RowArgs a;
    a.W = W; a.H = H; a.clamp = (float)s.alpha_clamp; a.cut = (float)s.alpha_cut;
    a.cutlo = (float)(s.alpha_cut * (1.0 - CUT_BAND)); a.cuthi = (float)(s.alpha_cut * (1.0 + CUT_BAND));
    a.clamp_d = s.alpha_clamp; a.cut_d = s.alpha_cut; a.degree = degree;
    a.iclamp = (float)(1.0 / s.alpha_clamp);
    for (int k = 0; k < 36; ++k) a.A[k] = A[k];
    for (int k = 0; k < 9; ++k) a.Rcw[k] = Rcw[k];
    if (m == 0) return cudaSuccess;
    const int64_t threads = m * 32;
    k_pose_rows<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(w, a, image, n_contrib, chain, ids, m, m_dev,
                                                                      rows);
    return cudaGetLastError();
}

cudaError_t launch_hb(const double* rows, const double* z, int64_t m, const int64_t* m_dev, double inv_s2, double* out,
                      double* part, cudaStream_t st) {
    k_hb_partial<<<HB_BLOCKS, 256, 0, st>>>(rows, z, m, m_dev, part);
    k_hb_final<<<1, 32 * HB_VALS, 0, st>>>(part, HB_BLOCKS, inv_s2, out);
    return cudaGetLastError();
}

int hb_scratch_doubles() { return HB_BLOCKS * HB_VALS; }

// Semi-dense selection + photometric residual + gate of the visual
// measurement on the device, no host round trip (estimator.py:241-277):
// ids = nonzero(mask) ascending; if more than `budget`, the ones at
// round(linspace(0, L-1, budget)) (numpy's k * step, half-to-even; the step
// exceeds 1 so the rounded indices are already unique); gray = channel mean
// ((r + g) + b) / 3 in f64; res = gray_obs - gray_hat, kept where |res| <=
// gate, in order.  counts = [L, selected, kept].
//   k_vs_count : per VS_CHUNK-pixel chunk, the number of mask hits
//   k_vs_emit  : the chunk's ascending ids at (sum of earlier chunks) + rank
//   k_vs_select: one CTA — subsample, residuals, gate, ordered compaction
constexpr int VS_THREADS = 256, VS_PER = 16, VS_CHUNK = VS_THREADS * VS_PER;

__device__ __forceinline__ int vs_block_scan(int v, int& total, int* s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    int before = 0, tot = 0;
    for (int k = 0; k < nw; ++k) {
        if (k < warp) before += s_w[k];
        tot += s_w[k];
    }
    total = tot;
    __syncthreads();
    return x - v + before;
}

__device__ __forceinline__ unsigned vs_bits(const uint8_t* mask, int64_t p0, int64_t npx) {
    unsigned bits = 0;
    if (p0 + VS_PER <= npx && ((uintptr_t)(mask + p0) & 15) == 0) {
        const uint4 q = *(const uint4*)(mask + p0);
        const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) bits |= (((w[i >> 2] >> (8 * (i & 3))) & 0xffu) != 0u) << i;
    } else {
        for (int i = 0; i < VS_PER; ++i)
            if (p0 + i < npx && mask[p0 + i]) bits |= 1u << i;
    }
    return bits;
}

__global__ void __launch_bounds__(VS_THREADS) k_vs_count(const uint8_t* __restrict__ mask, int64_t npx,
                                                          int* __restrict__ cnt) {
    __shared__ int s_w[VS_THREADS / 32];
    const int64_t p0 = (int64_t)blockIdx.x * VS_CHUNK + (int64_t)threadIdx.x * VS_PER;
    int tot;
    vs_block_scan(__popc(vs_bits(mask, p0, npx)), tot, s_w);
    if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(VS_THREADS) k_vs_emit(const uint8_t* __restrict__ mask, int64_t npx,
                                                         const int* __restrict__ cnt, int nchunk,
                                                         int32_t* __restrict__ ids_all, int* __restrict__ total) {
    __shared__ int s_w[VS_THREADS / 32];
    int before = 0, all;
    for (int k = threadIdx.x; k < nchunk; k += VS_THREADS) before += k < (int)blockIdx.x ? cnt[k] : 0;
    int dummy;
    const int ex = vs_block_scan(before, dummy, s_w);   // block sum of the earlier chunks
    (void)ex;
    const int64_t p0 = (int64_t)blockIdx.x * VS_CHUNK + (int64_t)threadIdx.x * VS_PER;
    unsigned bits = vs_bits(mask, p0, npx);
    int off = vs_block_scan(__popc(bits), all, s_w) + dummy;
    while (bits) {
        const int i = __ffs(bits) - 1;
        bits &= bits - 1;
        ids_all[off++] = (int32_t)(p0 + i);
    }
    if (blockIdx.x == nchunk - 1 && threadIdx.x == 0) *total = dummy + all;
}

__global__ void __launch_bounds__(1024) k_vs_select(const void* __restrict__ obs, bool u8, const float* __restrict__ img,
                                                    int budget, double gate, const int32_t* __restrict__ ids_all,
                                                    const int* __restrict__ total, int32_t* sel, double* sel_res,
                                                    int32_t* ids_out, double* res_out, int64_t* counts) {
    __shared__ int s_w[32];
    const int tid = threadIdx.x;
    const int L = *total;
    const int nsel = L > budget ? budget : L;
    const double step = budget > 1 ? (double)(L - 1) / (double)(budget - 1) : 0.0;
    for (int k = tid; k < nsel; k += 1024) {
        int src = k;
        if (L > budget) src = (budget > 1 && k == budget - 1) ? L - 1 : (int)rint((double)k * step);
        const int32_t p = ids_all[src];
        const float* h = img + 3 * (int64_t)p;
        const int64_t q = 3 * (int64_t)p;
        const double go = ((obs_value(obs, u8, q) + obs_value(obs, u8, q + 1)) + obs_value(obs, u8, q + 2)) / 3.0;
        const double gh = (((double)h[0] + (double)h[1]) + (double)h[2]) / 3.0;
        sel[k] = p;
        sel_res[k] = go - gh;
    }
    __syncthreads();
    const int per = (nsel + 1023) / 1024, c0 = tid * per;
    int c = 0;
    for (int j = 0; j < per; ++j)
        if (c0 + j < nsel && fabs(sel_res[c0 + j]) <= gate) ++c;
    int nok;
    int off = vs_block_scan(c, nok, s_w);
    for (int j = 0; j < per; ++j)
        if (c0 + j < nsel && fabs(sel_res[c0 + j]) <= gate) {
            ids_out[off] = sel[c0 + j];
            res_out[off] = sel_res[c0 + j];
            ++off;
        }
    if (tid == 0) {
        counts[0] = L;
        counts[1] = nsel;
        counts[2] = nok;
    }
}

int64_t visual_select_scratch_bytes(int64_t npx, int budget) {
    const int64_t nchunk = (npx + VS_CHUNK - 1) / VS_CHUNK;
    return 8 * ((nchunk + 1 + 1) / 2 + 1) + 4 * npx + 4 * (int64_t)budget + 8 + 8 * (int64_t)budget;
}

cudaError_t launch_visual_select(const uint8_t* mask, const void* obs, bool u8, const float* img, int64_t npx, int budget,
                                 double gate, void* scratch, int32_t* ids_out, double* res_out, int64_t* counts,
                                 cudaStream_t st) {
    const int nchunk = (int)((npx + VS_CHUNK - 1) / VS_CHUNK);
    int* cnt = (int*)scratch;                                          // nchunk + 1 (total)
    int* total = cnt + nchunk;
    int32_t* ids_all = (int32_t*)((char*)scratch + 8 * ((nchunk + 1 + 1) / 2 + 1));
    int32_t* sel = ids_all + npx;
    double* sel_res = (double*)(((uintptr_t)(sel + budget) + 7) & ~(uintptr_t)7);
    cudaError_t e = cudaMemsetAsync(total, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    if (nchunk > 0) {
        k_vs_count<<<nchunk, VS_THREADS, 0, st>>>(mask, npx, cnt);
        k_vs_emit<<<nchunk, VS_THREADS, 0, st>>>(mask, npx, cnt, nchunk, ids_all, total);
    }
    k_vs_select<<<1, 1024, 0, st>>>(obs, u8, img, budget, gate, ids_all, total, sel, sel_res, ids_out, res_out, counts);
    return cudaGetLastError();
}

cudaError_t launch_semidense(const void* obs, bool u8, const float* tfin, int W, int H, double thr, double tmax,
                             uint8_t* out, cudaStream_t st) {
    const dim3 grid((W + SD_BX - 1) / SD_BX, (H + SD_BY - 1) / SD_BY);
    k_semidense<<<grid, SD_BX * SD_BY, 0, st>>>(obs, u8, tfin, W, H, thr, tmax, out);
    return cudaGetLastError();
}

}  // namespace lsb
