// K3 blend forward and K4 blend backward: one CTA of 64 threads per 16x16
// tile, four horizontally adjacent pixels per thread (a warp owns an 8-row
// band), so each shared-memory record read feeds four pixel updates and the
// per-row terms (dy, E dy^2, s dy - mx) are computed once per thread.
//
// Records are staged into shared memory in batches of 64 (one 64 B record
// per thread, 16 B vector loads); all threads then read the same record
// (broadcast, conflict-free).  A warp whose 8-row band misses the splat's bbox
// skips it with one uniform test; inside the band every pixel applies the
// reference's per-pixel bbox membership test (exact CSR semantics,
// _kernels.py:21-59) before evaluating the exponential.
//
// The forward optionally fuses the photometric loss (optimize.py:48-74): the
// epilogue reads the observed pixels, writes dL/dI and reduces the loss sums
// per tile; the last CTA (ticket) adds the tile sums in tile order, so the
// value is deterministic.
//
// The backward recomputes the forward front to back per pixel and carries
// D = I - sum_{j<=k} w_j c_j, the suffix colour of the reference's
// back-to-front pass (_kernels.py:145-164); per (warp, splat) the 9 screen
// partials are reduced with a transpose-reduce (8 values in 16 shuffles + 1
// value in 5), summed over the two warps in shared memory and written once
// per (tile, splat) intersection — no global atomics, deterministic.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

constexpr int BT = 64;       // threads per tile CTA
constexpr int BATCH = 64;    // records per shared-memory batch
constexpr int PX = 4;        // pixels per thread (horizontal)

struct BlendArgs {
    int W, H;
    float clamp, tmin, cut;
    float bg0, bg1, bg2;
};

struct LossArgs {
    const float* observed;   // (H,W,3) or NULL: no fused loss
    float* grad;             // (H,W,3) dL/dI out
    double* sums;            // [ntiles*2] tile partials, then [2] totals at sums_out
    double* sums_out;
    unsigned long long* ticket;
    int kind;                // 0 L1, 1 L2
    float gscale;
};

__device__ __forceinline__ void stage_record(const Ws& w, int slot, int ox, int oy, float4* s_a, float4* s_b,
                                             float4* s_c, int t) {
    const Rec r = w.rec[slot];
    s_a[t] = make_float4((float)(r.mx - (double)ox), (float)(r.my - (double)oy), r.A, r.s);
    s_b[t] = make_float4(r.E, r.op, r.c0, r.c1);
    s_c[t] = make_float4(r.c2, r.z, __int_as_float(r.bbx), __int_as_float(r.bby));
}

template <bool DEPTH>
__global__ void __launch_bounds__(BT)
k_blend_fwd(Ws w, BlendArgs a, LossArgs L, float* __restrict__ image, float* __restrict__ t_final,
            int32_t* __restrict__ n_contrib, float* __restrict__ depth) {
    __shared__ float4 s_a[BATCH], s_b[BATCH], s_c[BATCH];
    __shared__ int s_last[BT / 32];
    __shared__ double s_loss[BT / 32][2];
    __shared__ bool s_final;
    const int tile = blockIdx.x;
    const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = tid >> 2, qx = (tid & 3) * PX;
    const int gy = oy + row, gx0 = ox + qx;
    const int wy0 = oy + warp * 8;
    const float fy = (float)row;
    float T[PX], cr[PX], cg[PX], cb[PX], dz[PX];
    int cnt[PX];
    unsigned done = 0;
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        T[j] = 1.f;
        cr[j] = cg[j] = cb[j] = dz[j] = 0.f;
        cnt[j] = 0;
        if (!(gy < a.H && gx0 + j < a.W)) done |= 1u << j;
    }
    int last = 0;
    const int start = w.tile_start[tile], end = w.tile_start[tile + 1];

    for (int base = start; base < end; base += BATCH) {
        if (__syncthreads_and(done == (1u << PX) - 1)) break;
        if (base + tid < end) stage_record(w, w.tile_slot[base + tid], ox, oy, s_a, s_b, s_c, tid);
        __syncthreads();
        const int nb = min(BATCH, end - base);
        for (int k = 0; k < nb; ++k) {
            const float4 qc = s_c[k];
            const int bby = __float_as_int(qc.w);
            const int y0 = bby & 0xffff, y1 = bby >> 16;
            if (y1 <= wy0 || y0 >= wy0 + 8) continue;                  // warp-uniform
            if (gy < y0 || gy >= y1) continue;                         // this thread's row
            const int bbx = __float_as_int(qc.z);
            const int lo = max((bbx & 0xffff) - gx0, 0), hi = min((bbx >> 16) - gx0, PX);
            if (lo >= hi) continue;
            const float4 qa = s_a[k], qb = s_b[k];
            const float dy = fy - qa.y;
            const float sdm = fmaf(qa.w, dy, -qa.x);      // u = x_local + s dy - mx
            const float edy = qb.x * dy * dy;
            bool used = false;
#pragma unroll
            for (int j = 0; j < PX; ++j) {
                if (j < lo || j >= hi || (done >> j) & 1u) continue;
                const float u = (float)(qx + j) + sdm;
                const float al = fminf(qb.y * ex2_approx(fmaf(qa.z, u * u, edy)), a.clamp);
                ++cnt[j];
                used = true;
                if (al >= a.cut) {
                    const float wt = T[j] * al;
                    cr[j] = fmaf(wt, qb.z, cr[j]);
                    cg[j] = fmaf(wt, qb.w, cg[j]);
                    cb[j] = fmaf(wt, qc.x, cb[j]);
                    if (DEPTH) dz[j] = fmaf(wt, qc.y, dz[j]);
                    T[j] = fmaf(-al, T[j], T[j]);
                    if (T[j] < a.tmin) done |= 1u << j;
                }
            }
            if (used) last = base + k + 1;
        }
    }
    // tile_last: how far into the list any pixel of the tile went
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (lane == 0) s_last[warp] = last;
    double l0 = 0.0, l1 = 0.0;
    if (gy < a.H) {
        const int64_t p0 = (int64_t)gy * a.W + gx0;
#pragma unroll
        for (int j = 0; j < PX; ++j) {
            if (gx0 + j >= a.W) break;
            const int64_t p = p0 + j;
            const float ir = cr[j] + T[j] * a.bg0, ig = cg[j] + T[j] * a.bg1, ib = cb[j] + T[j] * a.bg2;
            image[3 * p] = ir;
            image[3 * p + 1] = ig;
            image[3 * p + 2] = ib;
            t_final[p] = T[j];
            n_contrib[p] = cnt[j];
            if (DEPTH) depth[p] = dz[j];
            if (L.observed) {
                const float o3[3] = {L.observed[3 * p], L.observed[3 * p + 1], L.observed[3 * p + 2]};
                const float i3[3] = {ir, ig, ib};
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double d = (double)i3[c] - (double)o3[c];
                    l1 += d * d;
                    float gv;
                    if (L.kind == 0) {
                        l0 += fabs(d);
                        gv = d > 0.0 ? L.gscale : (d < 0.0 ? -L.gscale : 0.f);
                    } else {
                        l0 += d * d;
                        gv = (float)(2.0 * d * (double)L.gscale);
                    }
                    L.grad[3 * p + c] = gv;
                }
            }
        }
    }
    if (L.observed) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        if (lane == 0) {
            s_loss[warp][0] = l0;
            s_loss[warp][1] = l1;
        }
    }
    __syncthreads();
    if (tid == 0) {
        int m = start;
        for (int k = 0; k < BT / 32; ++k) m = max(m, s_last[k]);
        w.tile_last[tile] = m;
        if (L.observed) {
            L.sums[2 * tile] = s_loss[0][0] + s_loss[1][0];
            L.sums[2 * tile + 1] = s_loss[0][1] + s_loss[1][1];
            __threadfence();
            s_final = atomicAdd(L.ticket, 1ull) == gridDim.x - 1;
        }
    }
    if (!L.observed) return;
    __syncthreads();
    if (s_final) {
        __threadfence();
        // last CTA: deterministic sum of the tile partials, in tile order
        double v0 = 0.0, v1 = 0.0;
        for (int t = tid; t < (int)gridDim.x; t += BT) {
            v0 += ((volatile double*)L.sums)[2 * t];
            v1 += ((volatile double*)L.sums)[2 * t + 1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v0 += __shfl_xor_sync(0xffffffffu, v0, o);
            v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        }
        if (lane == 0) {
            s_loss[warp][0] = v0;
            s_loss[warp][1] = v1;
        }
        __syncthreads();
        if (tid == 0) {
            L.sums_out[0] = s_loss[0][0] + s_loss[1][0];
            L.sums_out[1] = s_loss[0][1] + s_loss[1][1];
            *L.ticket = 0;
        }
    }
}

// Transpose-reduce of v[0..7] across the warp: afterwards lane l holds the
// warp total of index ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 + ((l >> 2) & 1).
__device__ __forceinline__ float reduce8(float* v, int lane) {
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
    float a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = u16 ? v[i] : v[i + 4];
        const float keep = u16 ? v[i + 4] : v[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = u8 ? a[i] : a[i + 2];
        const float keep = u8 ? a[i + 2] : a[i];
        b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const float send = u4 ? b[0] : b[1];
    float c = (u4 ? b[1] : b[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    return c;
}

__global__ void __launch_bounds__(BT)
k_blend_bwd(Ws w, BlendArgs a, const float* __restrict__ image, const int32_t* __restrict__ n_contrib,
            const float* __restrict__ gimg, float gscale) {
    __shared__ float4 s_a[BATCH], s_b[BATCH], s_c[BATCH];
    __shared__ float2 s_d[BATCH];
    __shared__ float s_part[BT / 32][BATCH][NUM_PART];
    const int tile = blockIdx.x;
    const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = tid >> 2, qx = (tid & 3) * PX;
    const int gy = oy + row, gx0 = ox + qx;
    const int wy0 = oy + warp * 8;
    const float fy = (float)row;
    const float k2 = -2.0f / (float)LOG2E;     // undo the exp2 scaling: a_k = A k2, e = E k2
    // per-pixel state: T, D = I - prefix colour, dL/dI, entries left
    float T[PX], Dr[PX], Dg[PX], Db[PX], Gr[PX], Gg[PX], Gb[PX];
    int rem[PX];
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        T[j] = 1.f;
        Dr[j] = Dg[j] = Db[j] = Gr[j] = Gg[j] = Gb[j] = 0.f;
        rem[j] = 0;
        if (gy < a.H && gx0 + j < a.W) {
            const int64_t p = (int64_t)gy * a.W + gx0 + j;
            rem[j] = n_contrib[p];
            Dr[j] = image[3 * p];
            Dg[j] = image[3 * p + 1];
            Db[j] = image[3 * p + 2];
            Gr[j] = gimg[3 * p] * gscale;
            Gg[j] = gimg[3 * p + 1] * gscale;
            Gb[j] = gimg[3 * p + 2] * gscale;
        }
    }
    const int start = w.tile_start[tile], end = w.tile_last[tile];

    for (int base = start; base < end; base += BATCH) {
        bool alive = false;
#pragma unroll
        for (int j = 0; j < PX; ++j) alive |= rem[j] > 0;
        if (!__syncthreads_or(alive)) break;
        if (base + tid < end) {
            stage_record(w, w.tile_slot[base + tid], ox, oy, s_a, s_b, s_c, tid);
            s_d[tid] = make_float2(s_a[tid].z * k2, s_b[tid].x * k2);
        }
        __syncthreads();
        const int nb = min(BATCH, end - base);
        for (int k = 0; k < nb; ++k) {
            const float4 qc = s_c[k];
            const int bby = __float_as_int(qc.w);
            const int y0 = bby & 0xffff, y1 = bby >> 16;
            float acc[NUM_PART];
#pragma unroll
            for (int c = 0; c < NUM_PART; ++c) acc[c] = 0.f;
            bool any = false;
            if (!(y1 <= wy0 || y0 >= wy0 + 8) && gy >= y0 && gy < y1) {
                const int bbx = __float_as_int(qc.z);
                const int lo = max((bbx & 0xffff) - gx0, 0), hi = min((bbx >> 16) - gx0, PX);
                if (lo < hi) {
                    const float4 qa = s_a[k], qb = s_b[k];
                    const float2 qd = s_d[k];
                    const float dy = fy - qa.y;
                    const float sdm = fmaf(qa.w, dy, -qa.x);
                    const float edy = qb.x * dy * dy;
                    const float ey = qd.y * dy;
#pragma unroll
                    for (int j = 0; j < PX; ++j) {
                        if (j < lo || j >= hi || rem[j] <= 0) continue;
                        --rem[j];
                        any = true;
                        const float u = (float)(qx + j) + sdm;
                        const float G = ex2_approx(fmaf(qa.z, u * u, edy));
                        const float al = fminf(qb.y * G, a.clamp);
                        if (!(al >= a.cut) || al == 0.f) continue;
                        const float wt = T[j] * al;
                        Dr[j] = fmaf(-wt, qb.z, Dr[j]);
                        Dg[j] = fmaf(-wt, qb.w, Dg[j]);
                        Db[j] = fmaf(-wt, qc.x, Db[j]);
                        const float inv = rcp_approx(1.f - al);
                        const float da = Gr[j] * fmaf(qb.z, T[j], -Dr[j] * inv) +
                                         Gg[j] * fmaf(qb.w, T[j], -Dg[j] * inv) +
                                         Gb[j] * fmaf(qc.x, T[j], -Db[j] * inv);
                        acc[0] = fmaf(wt, Gr[j], acc[0]);
                        acc[1] = fmaf(wt, Gg[j], acc[1]);
                        acc[2] = fmaf(wt, Gb[j], acc[2]);
                        if (al < a.clamp) {
                            acc[3] = fmaf(G, da, acc[3]);
                            const float gq = qb.y * da * G;
                            const float v0 = qd.x * u;                 // (conic d)_x = a_k u
                            const float v1 = fmaf(qa.w, v0, ey);       // (conic d)_y = s v0 + e dy
                            acc[4] = fmaf(gq, v0, acc[4]);
                            acc[5] = fmaf(gq, v1, acc[5]);
                            const float hv0 = 0.5f * gq * v0;
                            acc[6] = fmaf(hv0, v0, acc[6]);
                            acc[7] = fmaf(hv0, v1, acc[7]);
                            acc[8] = fmaf(0.5f * gq * v1, v1, acc[8]);
                        }
                        T[j] = fmaf(-al, T[j], T[j]);
                    }
                }
            }
            if (__any_sync(0xffffffffu, any)) {
                const float r8 = reduce8(acc, lane);
                float r9 = acc[8];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) r9 += __shfl_xor_sync(0xffffffffu, r9, o);
                if ((lane & 3) == 0)
                    s_part[warp][k][((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1)] = r8;
                if (lane == 1) s_part[warp][k][8] = r9;
            } else if (lane < NUM_PART) {
                s_part[warp][k][lane] = 0.f;
            }
        }
        __syncthreads();
        if (tid < nb) {
            const int e = w.tile_e[base + tid];
            float* dst = w.part + (int64_t)e * NUM_PART;
#pragma unroll
            for (int c = 0; c < NUM_PART; ++c) dst[c] = s_part[0][tid][c] + s_part[1][tid][c];
        }
    }
    // intersections the walk never reached contribute nothing
    __syncthreads();
    const int fin = w.tile_start[tile + 1];
    for (int j = max(end, start) + tid; j < fin; j += BT) {
        float* dst = w.part + (int64_t)w.tile_e[j] * NUM_PART;
#pragma unroll
        for (int c = 0; c < NUM_PART; ++c) dst[c] = 0.f;
    }
}

cudaError_t launch_blend_fwd(const Ws& w, const lsb_settings& s, int W, int H, float* image, float* t_final,
                             int32_t* n_contrib, float* depth, const float* observed, int kind, float gscale,
                             float* grad, double* loss_out, cudaStream_t st) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2]};
    LossArgs L{observed, grad, w.loss_part, loss_out, w.ctr + 5, kind, gscale};
    if (depth)
        k_blend_fwd<true><<<w.ntiles, BT, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else
        k_blend_fwd<false><<<w.ntiles, BT, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    return cudaGetLastError();
}

cudaError_t launch_blend_bwd(const Ws& w, const lsb_settings& s, int W, int H, const float* image,
                             const int32_t* n_contrib, const float* gimg, float gscale, cudaStream_t st) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2]};
    k_blend_bwd<<<w.ntiles, BT, 0, st>>>(w, a, image, n_contrib, gimg, gscale);
    return cudaGetLastError();
}

}  // namespace lsb
