// K3 blend forward and K4 blend backward: one CTA per 16x16 tile.
//
// 128 threads per tile, two pixels per thread (rows r and r+2 of the warp's
// 4-row band), so every shared-memory record read feeds two pixel updates.
// Records are staged into shared memory in batches of 128 with 16-byte
// vector loads; every thread then walks the batch reading the same record
// (broadcast, conflict-free).  A warp whose 16x4 band misses the splat's bbox
// skips it with one uniform test; inside the band each pixel applies the
// reference's per-pixel bbox membership test (exact CSR semantics,
// _kernels.py:21-59) before evaluating the exponential.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

constexpr int BT = 128;      // threads per tile CTA
constexpr int BATCH = 128;   // records per shared-memory batch

struct BlendArgs {
    int W, H;
    float clamp, tmin, cut;
    float bg0, bg1, bg2;
};

__device__ __forceinline__ bool in_span(int v, int lo, int hi) {
    return (unsigned)(v - lo) < (unsigned)(hi - lo);
}

template <bool DEPTH>
__global__ void __launch_bounds__(BT)
k_blend_fwd(Ws w, BlendArgs a, float* __restrict__ image, float* __restrict__ t_final,
            int32_t* __restrict__ n_contrib, float* __restrict__ depth) {
    __shared__ float4 s_a[BATCH], s_b[BATCH], s_c[BATCH];
    __shared__ int s_last[BT / 32];
    const int tile = blockIdx.x;
    const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lx = lane & 15, ly0 = warp * 4 + (lane >> 4), ly1 = ly0 + 2;
    const int gx = ox + lx, gy0 = oy + ly0, gy1 = oy + ly1;
    const int wy0 = oy + warp * 4;
    const float fx = (float)lx, fy0 = (float)ly0, fy1 = (float)ly1;
    bool done0 = !(gx < a.W && gy0 < a.H), done1 = !(gx < a.W && gy1 < a.H);
    float T0 = 1.f, T1 = 1.f;
    float r0 = 0.f, g0 = 0.f, b0 = 0.f, d0 = 0.f, r1 = 0.f, g1 = 0.f, b1 = 0.f, d1 = 0.f;
    int cnt0 = 0, cnt1 = 0, last = 0;
    const int start = w.tile_start[tile], end = w.tile_start[tile + 1];

    for (int base = start; base < end; base += BATCH) {
        if (__syncthreads_and(done0 && done1)) break;
        const int j = base + tid;
        if (j < end) {
            const Rec r = w.rec[w.tile_slot[j]];
            s_a[tid] = make_float4((float)(r.mx - (double)ox), (float)(r.my - (double)oy), r.A, r.s);
            s_b[tid] = make_float4(r.E, r.op, r.c0, r.c1);
            s_c[tid] = make_float4(r.c2, r.z, __int_as_float(r.bbx), __int_as_float(r.bby));
        }
        __syncthreads();
        const int nb = min(BATCH, end - base);
        for (int k = 0; k < nb; ++k) {
            const float4 qc = s_c[k];
            const int bby = __float_as_int(qc.w);
            const int y0 = bby & 0xffff, y1 = bby >> 16;
            if (y1 <= wy0 || y0 >= wy0 + 4) continue;           // warp-uniform
            const int bbx = __float_as_int(qc.z);
            const int x0 = bbx & 0xffff, x1 = bbx >> 16;
            const bool inx = in_span(gx, x0, x1);
            const float4 qa = s_a[k], qb = s_b[k];
            const float ddx = fx - qa.x;
            if (!done0 && inx && in_span(gy0, y0, y1)) {
                const float dy = fy0 - qa.y;
                const float u = fmaf(qa.w, dy, ddx);
                const float al = fminf(qb.y * ex2_approx(fmaf(qa.z, u * u, qb.x * dy * dy)), a.clamp);
                ++cnt0;
                last = base + k + 1;
                if (al >= a.cut) {
                    const float wt = T0 * al;
                    r0 = fmaf(wt, qb.z, r0);
                    g0 = fmaf(wt, qb.w, g0);
                    b0 = fmaf(wt, qc.x, b0);
                    if (DEPTH) d0 = fmaf(wt, qc.y, d0);
                    T0 = fmaf(-al, T0, T0);
                    done0 = T0 < a.tmin;
                }
            }
            if (!done1 && inx && in_span(gy1, y0, y1)) {
                const float dy = fy1 - qa.y;
                const float u = fmaf(qa.w, dy, ddx);
                const float al = fminf(qb.y * ex2_approx(fmaf(qa.z, u * u, qb.x * dy * dy)), a.clamp);
                ++cnt1;
                last = base + k + 1;
                if (al >= a.cut) {
                    const float wt = T1 * al;
                    r1 = fmaf(wt, qb.z, r1);
                    g1 = fmaf(wt, qb.w, g1);
                    b1 = fmaf(wt, qc.x, b1);
                    if (DEPTH) d1 = fmaf(wt, qc.y, d1);
                    T1 = fmaf(-al, T1, T1);
                    done1 = T1 < a.tmin;
                }
            }
        }
    }
    // tile_last: how far into the list any pixel of the tile went
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (lane == 0) s_last[warp] = last;
    __syncthreads();
    if (tid == 0) {
        int m = start;
        for (int k = 0; k < BT / 32; ++k) m = max(m, s_last[k]);
        w.tile_last[tile] = m;
    }
    if (gx < a.W && gy0 < a.H) {
        const int64_t p = (int64_t)gy0 * a.W + gx;
        image[3 * p] = r0 + T0 * a.bg0;
        image[3 * p + 1] = g0 + T0 * a.bg1;
        image[3 * p + 2] = b0 + T0 * a.bg2;
        t_final[p] = T0;
        n_contrib[p] = cnt0;
        if (DEPTH) depth[p] = d0;
    }
    if (gx < a.W && gy1 < a.H) {
        const int64_t p = (int64_t)gy1 * a.W + gx;
        image[3 * p] = r1 + T1 * a.bg0;
        image[3 * p + 1] = g1 + T1 * a.bg1;
        image[3 * p + 2] = b1 + T1 * a.bg2;
        t_final[p] = T1;
        n_contrib[p] = cnt1;
        if (DEPTH) depth[p] = d1;
    }
}

// Per-pixel state of the backward walk (front-to-back recomputation).
struct BwdPix {
    float T, pr, pg, pb;     // transmittance, prefix colour sum_{j<=k} w_j c_j
    float ir, ig, ib;        // rendered pixel (image incl. background)
    float gr, gg, gb;        // dL/dI (scaled)
    int rem;                 // entries left to process (= forward n_contrib)
};

// One pixel's contribution to the 9 screen-space partials of one splat
// (_kernels.py:122-216 in forward order: S_k = I - P_k is the suffix colour).
__device__ __forceinline__ void bwd_pixel(BwdPix& s, const float4 qa, const float4 qb,
                                          const float4 qc, const float4 qd, float ddx, float dy,
                                          const BlendArgs& a, float* acc) {
    const float u = fmaf(qa.w, dy, ddx);
    const float G = ex2_approx(fmaf(qa.z, u * u, qb.x * dy * dy));
    const float al = fminf(qb.y * G, a.clamp);
    --s.rem;
    if (!(al >= a.cut) || al == 0.f) return;
    const float wt = s.T * al;
    s.pr = fmaf(wt, qb.z, s.pr);
    s.pg = fmaf(wt, qb.w, s.pg);
    s.pb = fmaf(wt, qc.x, s.pb);
    const float inv = 1.f / (1.f - al);
    const float da = s.gr * (qb.z * s.T - (s.ir - s.pr) * inv) +
                     s.gg * (qb.w * s.T - (s.ig - s.pg) * inv) +
                     s.gb * (qc.x * s.T - (s.ib - s.pb) * inv);
    acc[0] = fmaf(wt, s.gr, acc[0]);
    acc[1] = fmaf(wt, s.gg, acc[1]);
    acc[2] = fmaf(wt, s.gb, acc[2]);
    if (al < a.clamp) {
        acc[3] = fmaf(G, da, acc[3]);
        const float gq = qb.y * da * G;
        const float v0 = qd.x * u;                    // (conic d)_x = a_k u
        const float v1 = fmaf(qa.w, v0, qd.y * dy);   // (conic d)_y = s v0 + e dy
        acc[4] = fmaf(gq, v0, acc[4]);
        acc[5] = fmaf(gq, v1, acc[5]);
        const float hq = 0.5f * gq;
        acc[6] = fmaf(hq * v0, v0, acc[6]);
        acc[7] = fmaf(hq * v0, v1, acc[7]);
        acc[8] = fmaf(hq * v1, v1, acc[8]);
    }
    s.T = fmaf(-al, s.T, s.T);
}

__device__ __forceinline__ void load_pix(BwdPix& s, bool valid, int64_t p, const float* image,
                                         const int32_t* n_contrib, const float* gimg, float gs) {
    s.T = 1.f;
    s.pr = s.pg = s.pb = 0.f;
    s.rem = 0;
    s.ir = s.ig = s.ib = s.gr = s.gg = s.gb = 0.f;
    if (!valid) return;
    s.rem = n_contrib[p];
    s.ir = image[3 * p];
    s.ig = image[3 * p + 1];
    s.ib = image[3 * p + 2];
    s.gr = gimg[3 * p] * gs;
    s.gg = gimg[3 * p + 1] * gs;
    s.gb = gimg[3 * p + 2] * gs;
}

__global__ void __launch_bounds__(BT)
k_blend_bwd(Ws w, BlendArgs a, const float* __restrict__ image, const int32_t* __restrict__ n_contrib,
            const float* __restrict__ gimg, float gscale) {
    __shared__ float4 s_a[BATCH], s_b[BATCH], s_c[BATCH], s_d[BATCH];
    __shared__ float s_part[BT / 32][BATCH][NUM_PART];
    const int tile = blockIdx.x;
    const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lx = lane & 15, ly0 = warp * 4 + (lane >> 4), ly1 = ly0 + 2;
    const int gx = ox + lx, gy0 = oy + ly0, gy1 = oy + ly1;
    const int wy0 = oy + warp * 4;
    const float fx = (float)lx, fy0 = (float)ly0, fy1 = (float)ly1;
    BwdPix p0, p1;
    load_pix(p0, gx < a.W && gy0 < a.H, (int64_t)gy0 * a.W + gx, image, n_contrib, gimg, gscale);
    load_pix(p1, gx < a.W && gy1 < a.H, (int64_t)gy1 * a.W + gx, image, n_contrib, gimg, gscale);
    const int start = w.tile_start[tile], end = w.tile_last[tile];
    const float k2 = -2.0f / (float)LOG2E;   // undo the exp2 scaling: a_k = A * k2

    for (int base = start; base < end; base += BATCH) {
        if (__syncthreads_and(p0.rem <= 0 && p1.rem <= 0)) break;
        const int j = base + tid;
        if (j < end) {
            const Rec r = w.rec[w.tile_slot[j]];
            s_a[tid] = make_float4((float)(r.mx - (double)ox), (float)(r.my - (double)oy), r.A, r.s);
            s_b[tid] = make_float4(r.E, r.op, r.c0, r.c1);
            s_c[tid] = make_float4(r.c2, r.z, __int_as_float(r.bbx), __int_as_float(r.bby));
            s_d[tid] = make_float4(r.A * k2, r.E * k2, 0.f, 0.f);
        }
        __syncthreads();
        const int nb = min(BATCH, end - base);
        for (int k = 0; k < nb; ++k) {
            const float4 qc = s_c[k];
            const int bby = __float_as_int(qc.w);
            const int y0 = bby & 0xffff, y1 = bby >> 16;
            const bool band = !(y1 <= wy0 || y0 >= wy0 + 4);
            float acc[NUM_PART];
#pragma unroll
            for (int c = 0; c < NUM_PART; ++c) acc[c] = 0.f;
            bool any = false;
            if (band) {                                        // warp-uniform
                const int bbx = __float_as_int(qc.z);
                const int x0 = bbx & 0xffff, x1 = bbx >> 16;
                const bool inx = in_span(gx, x0, x1);
                const float4 qa = s_a[k], qb = s_b[k], qd = s_d[k];
                const float ddx = fx - qa.x;
                if (p0.rem > 0 && inx && in_span(gy0, y0, y1)) {
                    bwd_pixel(p0, qa, qb, qc, qd, ddx, fy0 - qa.y, a, acc);
                    any = true;
                }
                if (p1.rem > 0 && inx && in_span(gy1, y0, y1)) {
                    bwd_pixel(p1, qa, qb, qc, qd, ddx, fy1 - qa.y, a, acc);
                    any = true;
                }
            }
            if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                for (int c = 0; c < NUM_PART; ++c) {
                    float v = acc[c];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    acc[c] = v;
                }
                if (lane == 0) {
#pragma unroll
                    for (int c = 0; c < NUM_PART; ++c) s_part[warp][k][c] = acc[c];
                }
            } else if (lane < NUM_PART) {
                s_part[warp][k][lane] = 0.f;
            }
        }
        __syncthreads();
        if (tid < nb) {
            const int e = w.tile_e[base + tid];
#pragma unroll
            for (int c = 0; c < NUM_PART; ++c) {
                float v = s_part[0][tid][c];
#pragma unroll
                for (int q = 1; q < BT / 32; ++q) v += s_part[q][tid][c];
                w.part[(int64_t)c * w.cap + e] = v;
            }
        }
    }
    // entries the walk never reached contribute nothing
    __syncthreads();
    const int stop = end;
    const int fin = w.tile_start[tile + 1];
    for (int j = stop + tid; j < fin; j += BT) {
        const int e = w.tile_e[j];
#pragma unroll
        for (int c = 0; c < NUM_PART; ++c) w.part[(int64_t)c * w.cap + e] = 0.f;
    }
}

cudaError_t launch_blend_fwd(const Ws& w, const lsb_settings& s, int W, int H, float* image,
                             float* t_final, int32_t* n_contrib, float* depth, cudaStream_t st) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2]};
    if (depth)
        k_blend_fwd<true><<<w.ntiles, BT, 0, st>>>(w, a, image, t_final, n_contrib, depth);
    else
        k_blend_fwd<false><<<w.ntiles, BT, 0, st>>>(w, a, image, t_final, n_contrib, depth);
    return cudaGetLastError();
}

cudaError_t launch_blend_bwd(const Ws& w, const lsb_settings& s, int W, int H, const float* image,
                             const int32_t* n_contrib, const float* gimg, float gscale,
                             cudaStream_t st) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2]};
    k_blend_bwd<<<w.ntiles, BT, 0, st>>>(w, a, image, n_contrib, gimg, gscale);
    return cudaGetLastError();
}

}  // namespace lsb
