// K5 backward chain: one thread per visible splat (fixed grid, grid-stride).
//
// Takes the splat's summed per-intersection partials (k_chain_sums: a
// balanced, fixed-shape segmented reduction, so the result is
// deterministic), then applies the reference's chain rule
// in f64 (raster.py:267-399): 2-D covariance -> world covariance ->
// (rotation right tangent, scale); 2-D mean -> camera mean -> world mean;
// SH colour with the clamp gate and view-direction term; camera-tangent pose
// pieces reduced per block and finally by the last block (ticket), again in a
// fixed order.  Param gradients are accumulated (+=) into the N-shaped
// buffers, so multiple views add up in stream order without atomics.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

struct ChainArgs {
    lsb_params p;
    lsb_grads g;
    lsb_camera cam;
    lsb_pose T;
    int degree;
    double* pose_out;
};

__constant__ double c_SH2[16] = {
    0.28209479177387814, 0.4886025119029199, 1.0925484305920792, -1.0925484305920792,
    0.31539156525252005, -1.0925484305920792, 0.5462742152960396, -0.5900435899266435,
    2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
    1.445305721320277, -0.5900435899266435, 0.0, 0.0};

template <typename T>
__device__ void sh_basis_d(int degree, T x, T y, T z, T* b) {
    const double* C = c_SH2;
    b[0] = C[0];
    if (degree >= 1) { b[1] = -C[1] * y; b[2] = C[1] * z; b[3] = -C[1] * x; }
    if (degree >= 2) {
        const T xx = x * x, yy = y * y, zz = z * z;
        b[4] = C[2] * x * y; b[5] = C[3] * y * z; b[6] = C[4] * (2.0 * zz - xx - yy);
        b[7] = C[5] * x * z; b[8] = C[6] * (xx - yy);
        if (degree >= 3) {
            b[9] = C[7] * y * (3.0 * xx - yy); b[10] = C[8] * x * y * z;
            b[11] = C[9] * y * (4.0 * zz - xx - yy);
            b[12] = C[10] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            b[13] = C[11] * x * (4.0 * zz - xx - yy); b[14] = C[12] * z * (xx - yy);
            b[15] = C[13] * x * (xx - 3.0 * yy);
        }
    }
}

// d basis_k / d dir (sh.py:66-109), g[k][3].
template <typename T>
__device__ void sh_basis_grad_d(int degree, T x, T y, T z, T (*g)[3]) {
    const double* C = c_SH2;
    const int K = (degree + 1) * (degree + 1);
    for (int k = 0; k < K; ++k) g[k][0] = g[k][1] = g[k][2] = 0.0;
    if (degree >= 1) { g[1][1] = -C[1]; g[2][2] = C[1]; g[3][0] = -C[1]; }
    if (degree >= 2) {
        g[4][0] = C[2] * y; g[4][1] = C[2] * x;
        g[5][1] = C[3] * z; g[5][2] = C[3] * y;
        g[6][0] = C[4] * (-2.0 * x); g[6][1] = C[4] * (-2.0 * y); g[6][2] = C[4] * (4.0 * z);
        g[7][0] = C[5] * z; g[7][2] = C[5] * x;
        g[8][0] = C[6] * (2.0 * x); g[8][1] = C[6] * (-2.0 * y);
    }
    if (degree >= 3) {
        const T xx = x * x, yy = y * y, zz = z * z;
        g[9][0] = C[7] * 6.0 * x * y; g[9][1] = C[7] * (3.0 * xx - 3.0 * yy);
        g[10][0] = C[8] * y * z; g[10][1] = C[8] * x * z; g[10][2] = C[8] * x * y;
        g[11][0] = C[9] * (-2.0 * x * y); g[11][1] = C[9] * (4.0 * zz - xx - 3.0 * yy);
        g[11][2] = C[9] * (8.0 * y * z);
        g[12][0] = C[10] * (-6.0 * x * z); g[12][1] = C[10] * (-6.0 * y * z);
        g[12][2] = C[10] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
        g[13][0] = C[11] * (4.0 * zz - 3.0 * xx - yy); g[13][1] = C[11] * (-2.0 * x * y);
        g[13][2] = C[11] * (8.0 * x * z);
        g[14][0] = C[12] * (2.0 * x * z); g[14][1] = C[12] * (-2.0 * y * z); g[14][2] = C[12] * (xx - yy);
        g[15][0] = C[13] * (3.0 * xx - 3.0 * yy); g[15][1] = C[13] * (-6.0 * x * y);
    }
}

// ---- partial sums: a balanced segmented reduction over the intersections ----
// Intersections are splat-major (a splat's run is [vis_ebase[s],
// vis_ebase[s + 1]); emit_slot[e] names its splat).  One warp per chunk of
// CHAIN_CH = 128 intersections, lane l taking 4 consecutive ones (9 float4
// loads): each lane sums its runs locally in f64, then one segmented warp
// scan (fixed shape) stitches the runs that cross lanes.  A run closed inside
// the chunk is written back in f64 over its own first two partials (72 B of
// its own storage; a one-intersection run keeps its f32 partial); the
// chunk's first run when it started in an earlier chunk, and its last run
// when it continues in a later one, go to chain_carry[chunk] (first / last),
// which k_chain adds chunk by chunk in order.  Every sum has a fixed shape:
// deterministic, balanced however long a splat's run is, no atomics.
constexpr int CHAIN_PER_LANE = CHAIN_CH / 32;

__device__ __forceinline__ void store_f64x9(float* dst, const double* v) {
    uint32_t* d = (uint32_t*)dst;
#pragma unroll
    for (int c = 0; c < NUM_PART; ++c) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(v[c]);
        d[2 * c] = (uint32_t)b;
        d[2 * c + 1] = (uint32_t)(b >> 32);
    }
}

__device__ __forceinline__ double load_f64(const float* src, int c) {
    const uint32_t* s = (const uint32_t*)src;
    return __longlong_as_double((long long)(((unsigned long long)s[2 * c + 1] << 32) | s[2 * c]));
}

__global__ void __launch_bounds__(128) k_chain_sums(Ws w) {
    const int64_t I = (int64_t)w.ctr[1];
    if (I > (int64_t)w.cap) return;                  // overflow: no partials were written
    const int lane = threadIdx.x & 31;
    const int64_t nch = (I + CHAIN_CH - 1) / CHAIN_CH;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nch; c += nw) {
        const int64_t cb = c * CHAIN_CH, ce = cb + CHAIN_CH < I ? cb + CHAIN_CH : I;
        const int first_own = w.emit_slot[cb];
        const bool open_start = cb > 0 && w.emit_slot[cb - 1] == first_own;
        const int after_own = ce < I ? w.emit_slot[ce] : -3;
        double* carry = w.chain_carry + (size_t)c * 2 * NUM_PART;
        // ---- load the lane's 8 intersections ----
        const int64_t lb = cb + (int64_t)lane * CHAIN_PER_LANE;
        const int n = lb < ce ? (int)((ce - lb) < CHAIN_PER_LANE ? ce - lb : CHAIN_PER_LANE) : 0;
        float v[CHAIN_PER_LANE][NUM_PART];
        int own[CHAIN_PER_LANE];
        if (n == CHAIN_PER_LANE) {
            const float4* src = (const float4*)(w.part + lb * NUM_PART);
            float* dst = &v[0][0];
#pragma unroll
            for (int q = 0; q < CHAIN_PER_LANE * NUM_PART / 4; ++q) {
                const float4 x = __ldcs(src + q);
                dst[4 * q] = x.x;
                dst[4 * q + 1] = x.y;
                dst[4 * q + 2] = x.z;
                dst[4 * q + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < CHAIN_PER_LANE; ++k)
#pragma unroll
                for (int q = 0; q < NUM_PART; ++q) v[k][q] = k < n ? w.part[(lb + k) * NUM_PART + q] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < CHAIN_PER_LANE; ++k) own[k] = k < n ? w.emit_slot[lb + k] : -2;
        __syncwarp();                                  // every partial is read before any run is written back
        // ---- lane-local runs: head (first), closed interior ones, tail (last) ----
        double hs[NUM_PART], ts[NUM_PART];
#pragma unroll
        for (int q = 0; q < NUM_PART; ++q) hs[q] = ts[q] = 0.0;
        int nseg = 0, h_cnt = 0, t_cnt = 0;
        const int h_own = own[0];
        int t_own = -2;
        int64_t t_start = lb;
#pragma unroll
        for (int k = 0; k < CHAIN_PER_LANE; ++k) {
            if (k >= n) break;
            if (own[k] != t_own) {
                if (nseg == 1) {                       // the head closed inside the lane
#pragma unroll
                    for (int q = 0; q < NUM_PART; ++q) hs[q] = ts[q];
                    h_cnt = t_cnt;
                } else if (nseg >= 2 && t_cnt >= 2) {  // an interior run: closed, local
                    store_f64x9(w.part + t_start * NUM_PART, ts);
                }
                ++nseg;
                t_own = own[k];
                t_start = lb + k;
                t_cnt = 0;
#pragma unroll
                for (int q = 0; q < NUM_PART; ++q) ts[q] = 0.0;
            }
#pragma unroll
            for (int q = 0; q < NUM_PART; ++q) ts[q] += (double)v[k][q];
            ++t_cnt;
        }
        // ---- stitch the runs that cross lanes: segmented scan of the tails ----
        const int key = n ? t_own : -2 - lane;        // empty lanes: unique keys
        const int kup = __shfl_up_sync(0xffffffffu, key, 1);
        const int left_key = lane ? kup : (open_start ? first_own : -1);
        double S[NUM_PART];
#pragma unroll
        for (int q = 0; q < NUM_PART; ++q) S[q] = ts[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int ko = __shfl_up_sync(0xffffffffu, key, o);
            const bool add = lane >= o && ko == key;
#pragma unroll
            for (int q = 0; q < NUM_PART; ++q) {
                const double y = __shfl_up_sync(0xffffffffu, S[q], o);
                if (add) S[q] += y;
            }
        }
        double Sl[NUM_PART];                          // the scan at the lane to the left
#pragma unroll
        for (int q = 0; q < NUM_PART; ++q) Sl[q] = __shfl_up_sync(0xffffffffu, S[q], 1);
        const int right_head = __shfl_down_sync(0xffffffffu, n ? h_own : -7, 1);
        const bool last_lane = n > 0 && (lane == 31 || lb + n >= ce);
        // the head of a lane with >= 2 runs closes inside the lane
        if (n > 0 && nseg >= 2) {
            const bool cont = h_own == left_key;      // started in an earlier lane or chunk
            if (!cont) {
                if (h_cnt >= 2) store_f64x9(w.part + lb * NUM_PART, hs);
            } else {
                double tot[NUM_PART];
#pragma unroll
                for (int q = 0; q < NUM_PART; ++q) tot[q] = (lane ? Sl[q] : 0.0) + hs[q];
                if (h_own == first_own && open_start) {
#pragma unroll
                    for (int q = 0; q < NUM_PART; ++q) carry[q] = tot[q];       // chunk's first run: first
                } else {
                    store_f64x9(w.part + (int64_t)w.vis_ebase[h_own] * NUM_PART, tot);
                }
            }
        }
        // a lane's tail closes at the lane's end when the next lane starts another run
        if (n > 0 && (last_lane || right_head != t_own)) {
            const bool from_before = t_own == first_own && open_start;
            const bool open_end = last_lane && lb + n == ce && after_own == t_own;
            if (from_before)
#pragma unroll
                for (int q = 0; q < NUM_PART; ++q) carry[q] = S[q];
            if (open_end)
#pragma unroll
                for (int q = 0; q < NUM_PART; ++q) carry[NUM_PART + q] = S[q];
            if (!from_before && !open_end) {
                const bool cont = nseg == 1 && t_own == left_key;
                if (cont) store_f64x9(w.part + (int64_t)w.vis_ebase[t_own] * NUM_PART, S);
                else if (t_cnt >= 2) store_f64x9(w.part + t_start * NUM_PART, S);
            }
        }
        __syncwarp();
    }
}

using CT = double;  // chain-rule arithmetic: f64 keeps Adam's sign-sensitive first steps on the reference trajectory

// Parameter load from an f32 / f64 arena, widened to f64 (F64 fixed at compile time).
template <int F64>
__device__ __forceinline__ double tld(const void* p, int64_t i) {
    return F64 ? __ldg((const double*)p + i) : (double)__ldg((const float*)p + i);
}

// One thread per visible splat.  The thread's loads are issued in two waves
// (record header / intersection range / colour mask, then the splat's
// parameters, its current gradient rows and its partial sums together), so
// a splat costs two dependent memory round trips before its arithmetic
// instead of one per load; SH degree and arena dtype are template
// parameters, so the SH basis and its gradient stay in registers.
template <int DEG, int F64, bool POSE>
__global__ void __launch_bounds__(CHAIN_THREADS) k_chain(Ws w, ChainArgs a) {
    constexpr int KK = (DEG + 1) * (DEG + 1);
    __shared__ double s_red[CHAIN_THREADS / 32][POSE_VALS];
    __shared__ bool s_last;
    const int64_t M = (int64_t)w.ctr[0];
    CT R[9];
    for (int k = 0; k < 9; ++k) R[k] = (CT)a.T.R[k];
    double pose[POSE_VALS];
#pragma unroll
    for (int c = 0; c < POSE_VALS; ++c) pose[c] = 0.0;
    const int K = a.p.sh_coeffs;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; slot < M; slot += stride) {
        // ---- wave 1: the record header, the intersection range, the colour mask ----
        const int2 ie = *(const int2*)&w.rec[slot].id;           // id, ebase
        const int64_t e0 = w.vis_ebase[slot], e1 = w.vis_ebase[slot + 1];
        const uint32_t cm = w.colmask[slot];
        if (ie.y < 0 || e1 <= e0) continue;
        const int64_t i = ie.x;
        // ---- wave 2: parameters, gradient rows, partial sums ----
        const double px = tld<F64>(a.p.means, 3 * i), py = tld<F64>(a.p.means, 3 * i + 1),
                     pz = tld<F64>(a.p.means, 3 * i + 2);
        CT Rg[9], S[3];
#pragma unroll
        for (int k = 0; k < 9; ++k) Rg[k] = tld<F64>(a.p.rots, 9 * i + k);
#pragma unroll
        for (int k = 0; k < 3; ++k) S[k] = tld<F64>(a.p.scales, 3 * i + k);
        const int64_t sho = i * K * 3;
        CT shv[DEG >= 1 ? KK * 3 : 1];
        if (DEG >= 1) {
#pragma unroll
            for (int k = 0; k < KK * 3; ++k) shv[k] = tld<F64>(a.p.shs, sho + k);
        }
        float gm[3], gr[3], gs[3], gsh[KK * 3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            gm[k] = a.g.mean[3 * i + k];
            gr[k] = a.g.rot[3 * i + k];
            gs[k] = a.g.scale[3 * i + k];
        }
        const float go = a.g.opacity[i];
#pragma unroll
        for (int k = 0; k < KK * 3; ++k) gsh[k] = a.g.sh[sho + k];
        double q[NUM_PART];
        {
            const int64_t c0 = e0 / CHAIN_CH, c1 = (e1 - 1) / CHAIN_CH;
            if (c0 == c1) {
                const float* p = w.part + e0 * NUM_PART;
                if (e1 - e0 == 1) {
#pragma unroll
                    for (int k = 0; k < NUM_PART; ++k) q[k] = (double)p[k];
                } else {
#pragma unroll
                    for (int k = 0; k < NUM_PART; ++k) q[k] = load_f64(p, k);
                }
            } else {
                const double* cr = w.chain_carry;
#pragma unroll
                for (int k = 0; k < NUM_PART; ++k) q[k] = cr[(size_t)c0 * 2 * NUM_PART + NUM_PART + k];
                for (int64_t c = c0 + 1; c <= c1; ++c)
#pragma unroll
                    for (int k = 0; k < NUM_PART; ++k) q[k] += cr[(size_t)c * 2 * NUM_PART + k];
            }
        }
        bool nz = false;
#pragma unroll
        for (int c = 0; c < NUM_PART; ++c) nz |= (q[c] != 0.0);
        if (!nz) continue;
        // ---- recompute the forward geometry in f64 ----
        const CT x = (CT)(R[0] * px + R[1] * py + R[2] * pz + a.T.t[0]);
        const CT y = (CT)(R[3] * px + R[4] * py + R[5] * pz + a.T.t[1]);
        const CT z = (CT)(R[6] * px + R[7] * py + R[8] * pz + a.T.t[2]);
        const CT fx = a.cam.fx, fy = a.cam.fy;
        const CT J00 = fx / z, J02 = -fx * x / (z * z);
        const CT J11 = fy / z, J12 = -fy * y / (z * z);
        CT B[9], Wc[9];
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3) B[3 * r3 + c3] = Rg[3 * r3 + c3] * S[c3];
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3)
                Wc[3 * r3 + c3] = B[3 * r3] * B[3 * c3] + B[3 * r3 + 1] * B[3 * c3 + 1] +
                                  B[3 * r3 + 2] * B[3 * c3 + 2];
        CT Mm[6];   // M = J R (2x3)
        for (int k = 0; k < 3; ++k) {
            Mm[k] = J00 * R[k] + J02 * R[6 + k];
            Mm[3 + k] = J11 * R[3 + k] + J12 * R[6 + k];
        }
        // ---- 2-D covariance chain (raster.py:286-298) ----
        const CT S00 = q[6], S01 = q[7], S11 = q[8];
        CT SM[6];   // S M (2x3)
        for (int k = 0; k < 3; ++k) {
            SM[k] = S00 * Mm[k] + S01 * Mm[3 + k];
            SM[3 + k] = S01 * Mm[k] + S11 * Mm[3 + k];
        }
        CT dCw[9];  // M^T S M
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3) dCw[3 * r3 + c3] = Mm[r3] * SM[c3] + Mm[3 + r3] * SM[3 + c3];
        CT dM[6];   // 2 S M W
        for (int r2 = 0; r2 < 2; ++r2)
            for (int c3 = 0; c3 < 3; ++c3)
                dM[3 * r2 + c3] = 2.0f * (SM[3 * r2] * Wc[c3] + SM[3 * r2 + 1] * Wc[3 + c3] +
                                         SM[3 * r2 + 2] * Wc[6 + c3]);
        CT dJ[6];   // dM R^T
        for (int r2 = 0; r2 < 2; ++r2)
            for (int c3 = 0; c3 < 3; ++c3)
                dJ[3 * r2 + c3] = dM[3 * r2] * R[3 * c3] + dM[3 * r2 + 1] * R[3 * c3 + 1] +
                                  dM[3 * r2 + 2] * R[3 * c3 + 2];
        // d_W = J^T dM (3x3), J rows (J00,0,J02), (0,J11,J12)
        CT dW[9];
        for (int c3 = 0; c3 < 3; ++c3) {
            dW[c3] = J00 * dM[c3];
            dW[3 + c3] = J11 * dM[3 + c3];
            dW[6 + c3] = J02 * dM[c3] + J12 * dM[3 + c3];
        }
        // ---- mean chain ----
        const CT dm0 = q[4], dm1 = q[5];
        CT dmc[3] = {J00 * dm0, J11 * dm1, J02 * dm0 + J12 * dm1};
        const CT gxx = -fx / (z * z), gyy = -fy / (z * z);
        dmc[0] += dJ[2] * gxx;
        dmc[1] += dJ[5] * gyy;
        dmc[2] += dJ[0] * gxx + dJ[4] * gyy + dJ[2] * (2.0f * fx * x / (z * z * z)) +
                  dJ[5] * (2.0f * fy * y / (z * z * z));
        CT dmean[3];
        for (int k = 0; k < 3; ++k) dmean[k] = dmc[0] * R[k] + dmc[1] * R[3 + k] + dmc[2] * R[6 + k];
        // ---- covariance -> rotation tangent, scale ----
        CT dB[9];
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3)
                dB[3 * r3 + c3] = 2.0f * (dCw[3 * r3] * B[c3] + dCw[3 * r3 + 1] * B[3 + c3] +
                                         dCw[3 * r3 + 2] * B[6 + c3]);
        CT Y[9];   // Rg^T (dB * S)
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3)
                Y[3 * r3 + c3] = (Rg[r3] * dB[c3] + Rg[3 + r3] * dB[3 + c3] + Rg[6 + r3] * dB[6 + c3]) * S[c3];
        const CT drot[3] = {Y[7] - Y[5], Y[2] - Y[6], Y[3] - Y[1]};
        CT dscale[3];
        for (int c3 = 0; c3 < 3; ++c3)
            dscale[c3] = Rg[c3] * dB[c3] + Rg[3 + c3] * dB[3 + c3] + Rg[6 + c3] * dB[6 + c3];
        // ---- appearance ----
        const CT dcol[3] = {(cm & 1u) ? (CT)q[0] : 0.0f, (cm & 2u) ? (CT)q[1] : 0.0f, (cm & 4u) ? (CT)q[2] : 0.0f};
        const double* cc3 = a.T.cam_center;
        const CT dvx = px - cc3[0], dvy = py - cc3[1], dvz = pz - cc3[2];
        const CT dn = sqrt(dvx * dvx + dvy * dvy + dvz * dvz);
        CT dx_ = 0.0f, dy_ = 0.0f, dz_ = 1.0f;
        if (dn > 0.0f) {
            const CT inv = fmax(dn, 1e-30f);
            dx_ = dvx / inv; dy_ = dvy / inv; dz_ = dvz / inv;
        }
        CT b[16];
        sh_basis_d(DEG, dx_, dy_, dz_, b);
        float* gsho = a.g.sh + sho;
#pragma unroll
        for (int k = 0; k < KK; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) gsho[3 * k + c] = gsh[3 * k + c] + (float)(b[k] * dcol[c]);
        CT dpt[3] = {0.0f, 0.0f, 0.0f};
        if (DEG >= 1) {
            CT gb[16][3];
            sh_basis_grad_d(DEG, dx_, dy_, dz_, gb);
            CT dd[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int k = 0; k < KK; ++k) {
                const CT t = dcol[0] * shv[3 * k] + dcol[1] * shv[3 * k + 1] + dcol[2] * shv[3 * k + 2];
                dd[0] += t * gb[k][0]; dd[1] += t * gb[k][1]; dd[2] += t * gb[k][2];
            }
            const CT dot = dx_ * dd[0] + dy_ * dd[1] + dz_ * dd[2];
            const CT rr = fmax(dn, 1e-30f);
            dpt[0] = (dd[0] - dx_ * dot) / rr;
            dpt[1] = (dd[1] - dy_ * dot) / rr;
            dpt[2] = (dd[2] - dz_ * dot) / rr;
            dmean[0] += dpt[0]; dmean[1] += dpt[1]; dmean[2] += dpt[2];
        }
        // ---- write (accumulate) ----
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            a.g.mean[3 * i + k] = gm[k] + (float)dmean[k];
            a.g.rot[3 * i + k] = gr[k] + (float)drot[k];
            a.g.scale[3 * i + k] = gs[k] + (float)dscale[k];
        }
        a.g.opacity[i] = go + (float)q[3];
        if (!POSE) continue;       // the caller wants no pose gradient (window engine)
        // ---- pose pieces (camera tangent) ----
        CT Z[9];   // dW R^T
        for (int r3 = 0; r3 < 3; ++r3)
            for (int c3 = 0; c3 < 3; ++c3)
                Z[3 * r3 + c3] = dW[3 * r3] * R[3 * c3] + dW[3 * r3 + 1] * R[3 * c3 + 1] +
                                 dW[3 * r3 + 2] * R[3 * c3 + 2];
        pose[0] += y * dmc[2] - z * dmc[1] + (Z[7] - Z[5]);
        pose[1] += z * dmc[0] - x * dmc[2] + (Z[2] - Z[6]);
        pose[2] += x * dmc[1] - y * dmc[0] + (Z[3] - Z[1]);
        pose[3] += dmc[0];
        pose[4] += dmc[1];
        pose[5] += dmc[2];
        pose[6] -= dpt[0];
        pose[7] -= dpt[1];
        pose[8] -= dpt[2];
    }
    if (!POSE) return;
    // ---- deterministic pose reduction ----
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < POSE_VALS; ++c) {
        double v = pose[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_red[warp][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < POSE_VALS) {
        double v = 0.0;
        for (int k = 0; k < CHAIN_THREADS / 32; ++k) v += s_red[k][threadIdx.x];
        w.pose_part[blockIdx.x * POSE_VALS + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long t = atomicAdd(&w.ctr[4], 1ull);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {
        // all CHAIN_THREADS threads: thread t sums the blocks b = t, t + T, ...
        // (independent loads, pipelined), then a fixed tree over the threads
        __threadfence();
        double v[POSE_VALS];
#pragma unroll
        for (int c = 0; c < POSE_VALS; ++c) v[c] = 0.0;
        for (int b2 = threadIdx.x; b2 < (int)gridDim.x; b2 += CHAIN_THREADS)
#pragma unroll
            for (int c = 0; c < POSE_VALS; ++c) v[c] += __ldcg(w.pose_part + b2 * POSE_VALS + c);
#pragma unroll
        for (int c = 0; c < POSE_VALS; ++c) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
        }
        __syncthreads();
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < POSE_VALS; ++c) s_red[warp][c] = v[c];
        __syncthreads();
        if (threadIdx.x < POSE_VALS) {
            double t = 0.0;
            for (int k = 0; k < CHAIN_THREADS / 32; ++k) t += s_red[k][threadIdx.x];
            if (a.pose_out) a.pose_out[threadIdx.x] = t;
        }
        if (threadIdx.x == 0) w.ctr[4] = 0;
    }
}

template <int DEG, bool POSE>
static void chain_kernel_p(const Ws& w, const ChainArgs& a, cudaStream_t st) {
    if (a.p.dtype)
        k_chain<DEG, 1, POSE><<<CHAIN_BLOCKS, CHAIN_THREADS, 0, st>>>(w, a);
    else
        k_chain<DEG, 0, POSE><<<CHAIN_BLOCKS, CHAIN_THREADS, 0, st>>>(w, a);
}
template <int DEG>
static void chain_kernel(const Ws& w, const ChainArgs& a, cudaStream_t st) {
    if (a.pose_out)
        chain_kernel_p<DEG, true>(w, a, st);
    else
        chain_kernel_p<DEG, false>(w, a, st);
}

cudaError_t launch_chain(const Ws& w, const lsb_params& p, const lsb_grads& g, const lsb_camera& cam,
                         const lsb_pose& T, const lsb_settings& s, double* pose_out,
                         cudaStream_t st) {
    ChainArgs a{p, g, cam, T, 0, pose_out};
    int deg_store = 0;
    while ((deg_store + 2) * (deg_store + 2) <= p.sh_coeffs) ++deg_store;
    a.degree = s.sh_degree < deg_store ? s.sh_degree : deg_store;
    if (a.degree < 0) a.degree = 0;
    k_chain_sums<<<8 * 148, 128, 0, st>>>(w);
    switch (a.degree) {
        case 0: chain_kernel<0>(w, a, st); break;
        case 1: chain_kernel<1>(w, a, st); break;
        case 2: chain_kernel<2>(w, a, st); break;
        default: chain_kernel<3>(w, a, st); break;
    }
    return cudaGetLastError();
}

}  // namespace lsb
