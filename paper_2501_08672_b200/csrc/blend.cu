// K3 blend forward and K4 blend backward: ONE WARP per 16x16 tile (four
// independent tile-warps per CTA, no block barriers), eight pixels per lane
// (a 4-pixel horizontal run in rows r and r+8), so each shared-memory record
// read feeds eight pixel updates and the per-row terms (dy, E dy^2,
// s dy - mx) are computed once per row.
//
// The warp streams its tile's records through a double-buffered
// shared-memory slice: while it blends batch b (32 records, depth order,
// every lane reading the same record — broadcast, conflict-free), the copy
// engine path (cp.async, 4 x 16 B per record, no registers) is already
// fetching batch b+1, and the slot indices of batch b+2 are in flight.  Each pixel
// applies the reference's per-pixel bbox membership test (exact CSR
// semantics, _kernels.py:21-59) before it counts or blends an entry.
//
// Forward (_kernels.py:62-119): branch-free per pixel — alpha is evaluated
// for the whole 4-pixel run and masked, so no divergence inside the record
// loop.  Optionally fuses the photometric loss (optimize.py:48-74): the
// epilogue reads the observed pixels, writes dL/dI and reduces the loss per
// tile; the last CTA (ticket) adds the tile sums in tile order.
//
// Backward (_kernels.py:122-216): per pixel the forward is recomputed front
// to back, carrying T and gD = g . (I - sum_{j<=k} w_j c_j) — the dot product
// of dL/dI with the reference's suffix colour, updated as a scalar.  The 9
// screen partials of a (tile, splat) pair are reduced across the warp with a
// transpose-reduce and written once per intersection: no global atomics,
// deterministic.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

constexpr int WPB = 4;       // tile-warps per CTA
constexpr int RUN = 4;       // pixels per lane and row (horizontal run)
#ifndef FWD_MIN_BLOCKS
#define FWD_MIN_BLOCKS 6
#endif
#ifndef BWD_MIN_BLOCKS
#define BWD_MIN_BLOCKS 4
#endif

struct BlendArgs {
    int W, H;
    float clamp, tmin, cut;
    float bg0, bg1, bg2;
};

struct LossArgs {
    const float* observed;   // (H,W,3) or NULL: no fused loss
    float* grad;             // (H,W,3) dL/dI out
    double* sums;            // [ntiles*2] tile partials
    double* sums_out;        // [2] totals
    unsigned long long* ticket;
    int kind;                // 0 L1, 1 L2
    float gscale;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Per-warp record pipeline over one tile list [start, end).
struct RecPipe {
    Rec* buf;           // [2][32] in shared memory
    int start, end, slot_next;
    __device__ __forceinline__ void fetch(const Ws& w, int batch, int slot, int lane) {
        if (slot >= 0) {
            const float4* src = (const float4*)(w.rec + slot);
            float4* dst = (float4*)(buf + (batch & 1) * 32 + lane);
#pragma unroll
            for (int q = 0; q < 4; ++q) cp_async16(dst + q, src + q);
        }
        cp_commit();
    }
    __device__ __forceinline__ int slot_at(const Ws& w, int j) const { return j < end ? w.tile_slot[j] : -1; }
    // prologue: batch 0 in flight, slots of batch 1 loaded
    __device__ __forceinline__ void begin(const Ws& w, int lane) {
        fetch(w, 0, slot_at(w, start + lane), lane);
        slot_next = slot_at(w, start + 32 + lane);
    }
    // start fetching batch b+1, then wait for batch b; returns its records
    __device__ __forceinline__ const Rec* next(const Ws& w, int b, int lane) {
        fetch(w, b + 1, slot_next, lane);
        slot_next = slot_at(w, start + 32 * (b + 2) + lane);
        cp_wait<1>();
        __syncwarp();
        return buf + (b & 1) * 32;
    }
    __device__ __forceinline__ void drain() {
        cp_wait<0>();
        __syncwarp();
    }
};

template <bool DEPTH, bool CUT>
__global__ void __launch_bounds__(32 * WPB, FWD_MIN_BLOCKS)
k_blend_fwd(Ws w, BlendArgs a, LossArgs L, float* __restrict__ image, float* __restrict__ t_final,
            int32_t* __restrict__ n_contrib, float* __restrict__ depth) {
    __shared__ Rec s_rec[WPB][2 * 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int qx = (lane & 3) * RUN, r0 = lane >> 2;      // rows r0 and r0 + 8
    RecPipe pipe;
    pipe.buf = s_rec[wib];
    const float fx0 = (float)qx;
    const float fy[2] = {(float)r0, (float)(r0 + 8)};
    // persistent tile-warp: pull tiles from the queue until it is empty
    for (;;) {
        int tile = 0;
        if (lane == 0) tile = (int)atomicAdd(&w.ctr[7], 1ull);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= w.ntiles) break;
        const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
        const int gx0 = ox + qx;
        double l0 = 0.0, l1 = 0.0;
        // A pixel composites while T >= t_min (the reference breaks when
        // T < t_min, _kernels.py:98); pixels outside the image start at T = -1.
        float T[2][RUN], cr[2][RUN], cg[2][RUN], cb[2][RUN], dz[2][RUN];
        float cnt[2][RUN];     // processed-entry counts (exact in f32 below 2^24)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                T[h][j] = (oy + r0 + 8 * h < a.H && gx0 + j < a.W) ? 1.f : -1.f;
                cr[h][j] = cg[h][j] = cb[h][j] = dz[h][j] = 0.f;
                cnt[h][j] = 0.f;
            }
        int last = 0;
        const int start = w.tile_start[tile], end = w.tile_start[tile + 1];
        const float oxf = (float)ox, oyf = (float)oy;
        pipe.start = start;
        pipe.end = end;
        pipe.begin(w, lane);
        for (int b = 0, base = start; base < end; ++b, base += 32) {
            bool alive = false;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < RUN; ++j) alive |= T[h][j] >= a.tmin;
            if (!__any_sync(0xffffffffu, alive)) break;
            const Rec* sr = pipe.next(w, b, lane);
            const int nb = min(32, end - base);
            for (int k = 0; k < nb; ++k) {
                const int4 qi = *(const int4*)&sr[k].bbx;
                const int bby = qi.y, bbx = qi.x;
                const int y0 = (bby & 0xffff) - oy, y1 = (bby >> 16) - oy;
                const int lo = max((bbx & 0xffff) - gx0, 0), hi = min((bbx >> 16) - gx0, RUN);
                if (lo >= hi) continue;
                bool inx[RUN];                                       // bbox columns of this run
#pragma unroll
                for (int j = 0; j < RUN; ++j) inx[j] = j >= lo && j < hi;
                const float4 q0 = *(const float4*)&sr[k].mxh;        // mxh myh mxl myl
                const float4 qa = make_float4((q0.x - oxf) + q0.z, (q0.y - oyf) + q0.w, sr[k].A, sr[k].s);
                const float4 qb = *(const float4*)&sr[k].A;          // A s E op
                const float4 qc = *(const float4*)&sr[k].c0;         // c0 c1 c2 z
                const float lop = __log2f(qb.w);
                bool used = false;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int row = r0 + 8 * h;
                    if (row < y0 || row >= y1) continue;
                    const float dy = fy[h] - qa.y;
                    const float u0 = fmaf(qa.w, dy, fx0 - qa.x);      // u = x_local + s dy - mx
                    // log2(alpha) = A u^2 + E dy^2 + log2(op): opacity folded into the exponent
                    const float edy = fmaf(qb.z * dy, dy, lop);
#pragma unroll
                    for (int j = 0; j < RUN; ++j) {
                        const bool in = inx[j] && T[h][j] >= a.tmin;
                        const float u = j == 0 ? u0 : u0 + (float)j;
                        float al = fminf(ex2_approx(fmaf(qa.z, u * u, edy)), a.clamp);
                        cnt[h][j] += in ? 1.f : 0.f;
                        used |= in;
                        const bool take = CUT ? (in && al >= a.cut) : in;
                        al = take ? al : 0.f;
                        const float wt = T[h][j] * al;
                        cr[h][j] = fmaf(wt, qc.x, cr[h][j]);
                        cg[h][j] = fmaf(wt, qc.y, cg[h][j]);
                        cb[h][j] = fmaf(wt, qc.z, cb[h][j]);
                        if (DEPTH) dz[h][j] = fmaf(wt, qc.w, dz[h][j]);
                        T[h][j] = fmaf(-al, T[h][j], T[h][j]);
                    }
                }
                if (used) last = base + k + 1;
            }
            __syncwarp();
        }
        pipe.drain();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        if (lane == 0) w.tile_last[tile] = max(last, start);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gy = oy + r0 + 8 * h;
            if (gy >= a.H) continue;
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                if (gx0 + j >= a.W) continue;
                const int64_t p = (int64_t)gy * a.W + gx0 + j;
                const float ir = cr[h][j] + T[h][j] * a.bg0, ig = cg[h][j] + T[h][j] * a.bg1,
                            ib = cb[h][j] + T[h][j] * a.bg2;
                image[3 * p] = ir;
                image[3 * p + 1] = ig;
                image[3 * p + 2] = ib;
                t_final[p] = T[h][j];
                n_contrib[p] = (int32_t)cnt[h][j];
                if (DEPTH) depth[p] = dz[h][j];
                if (L.observed) {
                    const float i3[3] = {ir, ig, ib};
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double d = (double)i3[c] - (double)L.observed[3 * p + c];
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
        if (!L.observed) continue;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        unsigned long long done = 0;
        if (lane == 0) {
            L.sums[2 * tile] = l0;
            L.sums[2 * tile + 1] = l1;
            __threadfence();       // publish the tile partial before counting the tile done
            done = atomicAdd(L.ticket, 1ull);
        }
        done = __shfl_sync(0xffffffffu, done, 0);
        if (done != (unsigned long long)w.ntiles - 1) continue;
        // the warp that finished the last tile: deterministic sum in tile order
        __threadfence();
        double v0 = 0.0, v1 = 0.0;
        for (int t = lane; t < w.ntiles; t += 32) {
            v0 += ((volatile double*)L.sums)[2 * t];
            v1 += ((volatile double*)L.sums)[2 * t + 1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v0 += __shfl_xor_sync(0xffffffffu, v0, o);
            v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        }
        if (lane == 0) {
            L.sums_out[0] = v0;
            L.sums_out[1] = v1;
        }
    }
}

// Transpose-reduce of v[0..7] across the warp: afterwards lane l holds the
// warp total of index ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 + ((l >> 2) & 1).
__device__ __forceinline__ float reduce8(const float* v, int lane) {
    const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
    float a4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = u16 ? v[i] : v[i + 4];
        const float keep = u16 ? v[i + 4] : v[i];
        a4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float b2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = u8 ? a4[i] : a4[i + 2];
        const float keep = u8 ? a4[i + 2] : a4[i];
        b2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const float send = u4 ? b2[0] : b2[1];
    float c = (u4 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    return c;
}

__global__ void __launch_bounds__(32 * WPB, BWD_MIN_BLOCKS)
k_blend_bwd(Ws w, BlendArgs a, const float* __restrict__ image, const int32_t* __restrict__ n_contrib,
            const float* __restrict__ gimg, float gscale) {
    __shared__ Rec s_rec[WPB][2 * 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int qx = (lane & 3) * RUN, r0 = lane >> 2;
    const float k2 = -2.0f / (float)LOG2E;     // undo the exp2 scaling: a_k = A k2, e = E k2
    RecPipe pipe;
    pipe.buf = s_rec[wib];
    const float fx0 = (float)qx;
    const float fy[2] = {(float)r0, (float)(r0 + 8)};
    for (;;) {
        int tile = 0;
        if (lane == 0) tile = (int)atomicAdd(&w.ctr[8], 1ull);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= w.ntiles) break;
        const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
        const int gx0 = ox + qx;
        // per-pixel state: T, gD = g . (I - prefix colour), g = dL/dI, entries left
        float T[2][RUN], gD[2][RUN], Gr[2][RUN], Gg[2][RUN], Gb[2][RUN];
        int rem[2][RUN];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                T[h][j] = 1.f;
                gD[h][j] = Gr[h][j] = Gg[h][j] = Gb[h][j] = 0.f;
                rem[h][j] = 0;
                const int gy = oy + r0 + 8 * h;
                if (gy < a.H && gx0 + j < a.W) {
                    const int64_t p = (int64_t)gy * a.W + gx0 + j;
                    rem[h][j] = n_contrib[p];
                    Gr[h][j] = gimg[3 * p] * gscale;
                    Gg[h][j] = gimg[3 * p + 1] * gscale;
                    Gb[h][j] = gimg[3 * p + 2] * gscale;
                    gD[h][j] = Gr[h][j] * image[3 * p] + Gg[h][j] * image[3 * p + 1] + Gb[h][j] * image[3 * p + 2];
                }
            }
        const int start = w.tile_start[tile], end = w.tile_last[tile];
        const float oxf = (float)ox, oyf = (float)oy;
        pipe.start = start;
        pipe.end = end;
        pipe.begin(w, lane);
        for (int b = 0, base = start; base < end; ++b, base += 32) {
            bool alive = false;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < RUN; ++j) alive |= rem[h][j] > 0;
            if (!__any_sync(0xffffffffu, alive)) break;
            const Rec* sr = pipe.next(w, b, lane);
            const int nb = min(32, end - base);
            for (int k = 0; k < nb; ++k) {
                const float4 q0 = *(const float4*)&sr[k].mxh;        // mxh myh mxl myl
                const float4 q1 = *(const float4*)&sr[k].A;          // A s E op
                const float4 q2 = *(const float4*)&sr[k].c0;         // c0 c1 c2 z
                const int4 q3 = *(const int4*)&sr[k].bbx;            // bbx bby id ebase
                // record in the (mx, my, A, s) (E, op, c0, c1) (c2, z) layout the math below uses
                const float4 qa = make_float4((q0.x - oxf) + q0.z, (q0.y - oyf) + q0.w, q1.x, q1.y);
                const float4 qb = make_float4(q1.z, q1.w, q2.x, q2.y);
                const float4 qc = make_float4(q2.z, q2.w, 0.f, 0.f);
                const float2 qd = make_float2(q1.x * k2, q1.z * k2);
                const int bby = q3.y, bbx = q3.x;
                const int y0 = (bby & 0xffff) - oy, y1 = (bby >> 16) - oy;
                const int lo = max((bbx & 0xffff) - gx0, 0), hi = min((bbx >> 16) - gx0, RUN);
                bool inx[RUN];
#pragma unroll
                for (int j = 0; j < RUN; ++j) inx[j] = j >= lo && j < hi;
                // accumulators: colour (3), sum gd, sum gd v0, sum gd v1, sum gd v0^2,
                // sum gd v0 v1, sum gd v1^2 with gd = G dalpha and v = conic d
                // (op is factored out and applied once per record below)
                float acc[9];
#pragma unroll
                for (int c = 0; c < 9; ++c) acc[c] = 0.f;
                bool any = false;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int row = r0 + 8 * h;
                    if (row < y0 || row >= y1 || lo >= hi) continue;
                    const float dy = fy[h] - qa.y;
                    const float u0 = fmaf(qa.w, dy, fx0 - qa.x);
                    const float edy = qb.x * dy * dy;
                    const float ey = qd.y * dy;
                    // branch-free per pixel: entries outside the bbox, past the
                    // pixel's processed count, or below alpha_cut get alpha = 0,
                    // which leaves T, gD and every accumulator unchanged
#pragma unroll
                    for (int j = 0; j < RUN; ++j) {
                        const bool in = inx[j] && rem[h][j] > 0;
                        rem[h][j] -= in ? 1 : 0;
                        any |= in;
                        const float u = j == 0 ? u0 : u0 + (float)j;
                        const float G = ex2_approx(fmaf(qa.z, u * u, edy));
                        const float al0 = fminf(qb.y * G, a.clamp);
                        const bool take = in && al0 >= a.cut;
                        const float al = take ? al0 : 0.f;
                        const float t = T[h][j];
                        const float wt = t * al;
                        const float gc = fmaf(Gr[h][j], qb.z, fmaf(Gg[h][j], qb.w, Gb[h][j] * qc.x));
                        gD[h][j] = fmaf(-wt, gc, gD[h][j]);               // g . suffix colour after k
                        const float da = fmaf(t, gc, -gD[h][j] * rcp_approx(1.f - al));
                        acc[0] = fmaf(wt, Gr[h][j], acc[0]);
                        acc[1] = fmaf(wt, Gg[h][j], acc[1]);
                        acc[2] = fmaf(wt, Gb[h][j], acc[2]);
                        // clamp gate (_kernels.py:201): saturated alpha passes no geometry gradient
                        const float gd = (take && al < a.clamp) ? G * da : 0.f;
                        const float v0 = qd.x * u;                  // (conic d)_x = a_k u
                        const float v1 = fmaf(qa.w, v0, ey);        // (conic d)_y = s v0 + e dy
                        const float g0 = gd * v0, g1 = gd * v1;
                        acc[3] += gd;
                        acc[4] += g0;
                        acc[5] += g1;
                        acc[6] = fmaf(g0, v0, acc[6]);
                        acc[7] = fmaf(g0, v1, acc[7]);
                        acc[8] = fmaf(g1, v1, acc[8]);
                        T[h][j] = fmaf(-al, t, t);
                    }
                }
                float val = 0.f;
                if (__any_sync(0xffffffffu, any)) {
                    // index i of the 8-vector lands in lanes 4i..4i+3 (reduce8)
                    const float r8 = reduce8(acc, lane);
                    float r9 = acc[8];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) r9 += __shfl_xor_sync(0xffffffffu, r9, o);
                    val = __shfl_sync(0xffffffffu, r8, 4 * min(lane, 7));
                    if (lane == 8) val = r9;
                    const float op = qb.y;
                    val *= (lane < 4) ? 1.f : ((lane < 6) ? op : 0.5f * op);
                }
                if (lane < NUM_PART) w.part[(int64_t)w.tile_e[base + k] * NUM_PART + lane] = val;
            }
            __syncwarp();
        }
        pipe.drain();
        // intersections the walk never reached contribute nothing
        const int fin = w.tile_start[tile + 1];
        for (int j = max(end, start); j < fin; ++j)
            if (lane < NUM_PART) w.part[(int64_t)w.tile_e[j] * NUM_PART + lane] = 0.f;
    }
}

// CTAs to launch for a persistent tile-warp kernel: every resident slot once.
static int persistent_grid(const void* fn, int ntiles) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * WPB, 0);
    const int need = (ntiles + WPB - 1) / WPB;
    const int g = sms * (per_sm > 0 ? per_sm : 1);
    return g < need ? g : need;
}

cudaError_t launch_blend_fwd(const Ws& w, const lsb_settings& s, int W, int H, float* image, float* t_final,
                             int32_t* n_contrib, float* depth, const float* observed, int kind, float gscale,
                             float* grad, double* loss_out, cudaStream_t st) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2]};
    LossArgs L{observed, grad, w.loss_part, loss_out, w.ctr + 5, kind, gscale};
    // reset the loss done-count and the forward tile queue ([5], [7])
    cudaError_t e = cudaMemsetAsync(w.ctr + 5, 0, 3 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const bool cut = s.alpha_cut > 0.0;
    const int grid = persistent_grid(depth ? (cut ? (const void*)k_blend_fwd<true, true> : (const void*)k_blend_fwd<true, false>)
                                           : (cut ? (const void*)k_blend_fwd<false, true> : (const void*)k_blend_fwd<false, false>),
                                     w.ntiles);
    if (depth && cut)
        k_blend_fwd<true, true><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else if (depth)
        k_blend_fwd<true, false><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else if (cut)
        k_blend_fwd<false, true><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else
        k_blend_fwd<false, false><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    return cudaGetLastError();
}

cudaError_t launch_blend_bwd(const Ws& w, const lsb_settings& s, int W, int H, const float* image,
                             const int32_t* n_contrib, const float* gimg, float gscale, cudaStream_t st) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2]};
    cudaError_t e = cudaMemsetAsync(w.ctr + 8, 0, sizeof(unsigned long long), st);   // backward tile queue
    if (e != cudaSuccess) return e;
    k_blend_bwd<<<persistent_grid((const void*)k_blend_bwd, w.ntiles), 32 * WPB, 0, st>>>(w, a, image, n_contrib,
                                                                                         gimg, gscale);
    return cudaGetLastError();
}

}  // namespace lsb
