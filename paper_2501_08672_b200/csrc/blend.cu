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
// Issue budget.  The inner loops are bound by instruction issue, and the ALU
// pipe (compares, selects, min/max — half rate on this SM) was the hot one,
// so per (pixel, splat) pair the code keeps ALU work to the two predicates
// the semantics need (alive-and-in-bbox, alpha >= cut) and puts everything
// else on the FMA pipe: the alpha clamp is a saturate (alpha = clamp * sat(
// op g / clamp), 1/clamp folded into the exponent and clamp into the
// colours), and the gated updates are predicated instead of selected.
//
// Saturation is only possible for a record whose opacity reaches the clamp
// (op g / clamp >= 1 needs lop = log2(op / clamp) >= 0), so the backward picks
// per record, warp-uniformly, a path with or without the saturate and the
// a < 1 gate: for lop < -1e-6 the two paths give the same bits.
//
// Forward (_kernels.py:62-119): alpha is evaluated for the whole 4-pixel run
// and the updates are predicated, so there is no divergence inside the
// record loop.  Without a processed-entry count (n_contrib == NULL, the
// window engine) the count update is dropped.  Optionally fuses the photometric loss (optimize.py:48-74): the
// epilogue reads the observed pixels, writes dL/dI and reduces the loss per
// tile; k_loss_total then adds the tile sums in a fixed order.
//
// Backward (_kernels.py:122-216): per pixel the forward is recomputed front
// to back with the SAME instruction sequence (shared helpers below), so T is
// bit-identical to the forward's and a pixel stops exactly where it stopped
// there (T < t_min) without a per-pixel entry count.  It carries T and
// gD = g . (I - sum_{j<=k} w_j c_j) — the dot product of dL/dI with the
// reference's suffix colour, updated as a scalar.  Per row the geometric
// terms are accumulated as raw moments of (u, dy) (sum gd, gd u, gd u^2) and
// mapped to the conic-space sums once per record; the 9 screen partials of
// a (tile, splat) pair are reduced across the warp with a transpose-reduce
// and written once per intersection: no global atomics, deterministic.
#include <cuda_runtime.h>

#include "common.cuh"

namespace lsb {

#ifndef LSB_WPB
#define LSB_WPB 4
#endif
#ifndef LSB_BLEND_PRIO
#define LSB_BLEND_PRIO 0      // launch the fused blend at the greatest priority (cudaLaunchAttributePriority)
#endif
#ifndef FUSED_RESERVE
#define FUSED_RESERVE 1      // CTA slots per SM the fused blend leaves to the other lanes
#endif
constexpr int WPB = LSB_WPB;  // tile-warps per CTA
constexpr int RUN = RUN_PX;  // pixels per lane and row (horizontal run)
#ifndef FWD_MIN_BLOCKS
#define FWD_MIN_BLOCKS 6
#endif
#ifndef BWD_MIN_BLOCKS
#define BWD_MIN_BLOCKS 5
#endif
#ifndef BWD_UNROLL
#define BWD_UNROLL 1          // record-loop unroll of the backward walk
#endif
#ifndef FUSED_FWD_UNROLL
#define FUSED_FWD_UNROLL 1    // record-loop unroll of the fused kernel's forward walk
#endif
constexpr int kBwdUnroll = BWD_UNROLL, kFusedFwdUnroll = FUSED_FWD_UNROLL;

struct BlendArgs {
    int W, H;
    float clamp, tmin, cut;
    float bg0, bg1, bg2;
    float cutp;       // cut / clamp: the test on the saturated alpha
    float ik;         // 1 / clamp
    float cutlo, cuthi;    // cut' (1 -+ CUT_BAND): the band where a flagged entry's pairs are decided in f64
    double clamp_d, cut_d;
    float bflim;           // records with lop <= bflim are bbox-free (common.cuh bbox_free_lim)
};

// Per-column liveness threshold of a record: T must reach t_min for pixels
// inside the bbox columns [cx0, cx1) of the run, +inf outside, so one
// compare gives "alive and in bbox".
__device__ __forceinline__ float col_thr(int j, int cx0, int cx1, float tmin) {
    return (j >= cx0 && j < cx1) ? tmin : __int_as_float(0x7f800000);
}

// ---- the alpha_cut band -----------------------------------------------------
// The walks decide `alpha < alpha_cut` (_kernels.py:104) in f32.  Where the
// f32 alpha lies too close to the cut for that to be the reference's f64
// decision, the decision was taken in f64 during binning (preprocess.cu,
// band_search in the scatter): a tile entry with such pixels carries OVR_BIT
// in tile_slot and a row of 256-bit masks (the tile's band pixels, and their
// f64 decisions), which the walks' threshold for those pixels follows: 0
// (composite) or +inf (skip) instead of cut'.  All other pairs are decided in
// f32 at least 5x farther from the cut than the f32 alpha's error (CUT_BAND,
// common.cuh); the hot path pays one bit test per record.

// Thresholds of the lane's pixels for a flagged entry.  Nibble h holds the
// lane's 4 pixels of row r0 + 8h.
struct OvrNib {
    unsigned band[2], take[2];
};
__device__ __forceinline__ OvrNib ovr_nibbles(const Ws& w, int j, int lane) {
    const uint32_t* m = w.ovr + (size_t)w.ovr_of[w.tile_e[j]] * 16;
    OvrNib o;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int bit = ((lane >> 2) + 8 * h) * TILE + (lane & 3) * RUN;
        o.band[h] = (m[bit >> 5] >> (bit & 31)) & 0xfu;
        o.take[h] = (m[8 + (bit >> 5)] >> (bit & 31)) & 0xfu;
    }
    return o;
}
__device__ __forceinline__ float ovr_cut(const OvrNib& o, int h, int j, float cutp) {
    return ((o.band[h] >> j) & 1u) ? (((o.take[h] >> j) & 1u) ? 0.f : __int_as_float(0x7f800000)) : cutp;
}

// Forward pixel update, predicated (no branches, no selects):
//   in   = T >= thr            (alive and inside the bbox)   -> count
//   take = in && a >= cut'                                    -> composite
//   w = T a;  C += w c';  T += w (-clamp)
__device__ __forceinline__ void fwd_pixel(float al, float thr, float cutp, float nkap, float c0, float c1, float c2,
                                          float& T, float& cnt, float& cr, float& cg, float& cb) {
    asm("{\n\t.reg .pred pi, pt;\n\t.reg .f32 w;\n\t"
        "setp.ge.f32 pi, %0, %5;\n\t"
        "@pi add.f32 %1, %1, 0f3F800000;\n\t"
        "setp.ge.and.f32 pt, %6, %7, pi;\n\t"
        "mul.rn.f32 w, %0, %6;\n\t"
        "@pt fma.rn.f32 %2, w, %8, %2;\n\t"
        "@pt fma.rn.f32 %3, w, %9, %3;\n\t"
        "@pt fma.rn.f32 %4, w, %10, %4;\n\t"
        "@pt fma.rn.f32 %0, w, %11, %0;\n\t}"
        : "+f"(T), "+f"(cnt), "+f"(cr), "+f"(cg), "+f"(cb)
        : "f"(thr), "f"(al), "f"(cutp), "f"(c0), "f"(c1), "f"(c2), "f"(nkap));
}

// Forward pixel update without the entry count (same T recurrence):
//   take = T >= thr && a >= cut'  ->  w = T a;  C += w c';  T += w (-clamp)
__device__ __forceinline__ void fwd_pixel_nc(float al, float thr, float cutp, float nkap, float c0, float c1, float c2,
                                             float& T, float& cr, float& cg, float& cb) {
    asm("{\n\t.reg .pred pi, pt;\n\t.reg .f32 w;\n\t"
        "setp.ge.f32 pi, %0, %4;\n\t"
        "setp.ge.and.f32 pt, %5, %6, pi;\n\t"
        "mul.rn.f32 w, %0, %5;\n\t"
        "@pt fma.rn.f32 %1, w, %7, %1;\n\t"
        "@pt fma.rn.f32 %2, w, %8, %2;\n\t"
        "@pt fma.rn.f32 %3, w, %9, %3;\n\t"
        "@pt fma.rn.f32 %0, w, %10, %0;\n\t}"
        : "+f"(T), "+f"(cr), "+f"(cg), "+f"(cb)
        : "f"(thr), "f"(al), "f"(cutp), "f"(c0), "f"(c1), "f"(c2), "f"(nkap));
}

__device__ __forceinline__ void fwd_pixel_depth(float al, float thr, float cutp, float nkap, float c0, float c1,
                                                float c2, float zk, float& T, float& cnt, float& cr, float& cg,
                                                float& cb, float& dz) {
    asm("{\n\t.reg .pred pi, pt;\n\t.reg .f32 w;\n\t"
        "setp.ge.f32 pi, %0, %6;\n\t"
        "@pi add.f32 %1, %1, 0f3F800000;\n\t"
        "setp.ge.and.f32 pt, %7, %8, pi;\n\t"
        "mul.rn.f32 w, %0, %7;\n\t"
        "@pt fma.rn.f32 %2, w, %9, %2;\n\t"
        "@pt fma.rn.f32 %3, w, %10, %3;\n\t"
        "@pt fma.rn.f32 %4, w, %11, %4;\n\t"
        "@pt fma.rn.f32 %5, w, %12, %5;\n\t"
        "@pt fma.rn.f32 %0, w, %13, %0;\n\t}"
        : "+f"(T), "+f"(cnt), "+f"(cr), "+f"(cg), "+f"(cb), "+f"(dz)
        : "f"(thr), "f"(al), "f"(cutp), "f"(c0), "f"(c1), "f"(c2), "f"(zk), "f"(nkap));
}

// Backward pixel update (same T recurrence as fwd_pixel), predicated:
//   take: w = T a; gc' = g.c'; gD -= w gc'; dap = T gc' - gD / (1/clamp - a);
//         colour sums += w g; T += w (-clamp)
//   gate = take && a < 1 (unclamped): gd = a dap; S0 += gd; S1 += gd u; S2 += gd u^2
// Without SAT the record cannot saturate and gate == take.
#define LSB_BWD_BODY(GATE_SETP, GP)                                         \
    "{\n\t.reg .pred pi, pt, pg;\n\t.reg .f32 w, gc, r, tg, da, gd, gu;\n\t" \
    "setp.ge.f32 pi, %0, %8;\n\t"                                           \
    "setp.ge.and.f32 pt, %9, %10, pi;\n\t" GATE_SETP                        \
    "mul.rn.f32 w, %0, %9;\n\t"                                             \
    "mul.rn.f32 gc, %20, %15;\n\t"                                          \
    "fma.rn.f32 gc, %19, %14, gc;\n\t"                                      \
    "fma.rn.f32 gc, %18, %13, gc;\n\t"                                      \
    "neg.f32 r, w;\n\t"                                                     \
    "@pt fma.rn.f32 %1, r, gc, %1;\n\t"                                     \
    "sub.f32 r, %12, %9;\n\t"                                               \
    "rcp.approx.ftz.f32 r, r;\n\t"                                          \
    "mul.rn.f32 tg, %0, gc;\n\t"                                            \
    "neg.f32 da, %1;\n\t"                                                   \
    "fma.rn.f32 da, da, r, tg;\n\t"                                         \
    "@pt fma.rn.f32 %2, w, %18, %2;\n\t"                                    \
    "@pt fma.rn.f32 %3, w, %19, %3;\n\t"                                    \
    "@pt fma.rn.f32 %4, w, %20, %4;\n\t"                                    \
    "mul.rn.f32 gd, %9, da;\n\t"                                            \
    "mul.rn.f32 gu, gd, %16;\n\t"                                           \
    "@" GP " add.f32 %5, %5, gd;\n\t"                                       \
    "@" GP " add.f32 %6, %6, gu;\n\t"                                       \
    "@" GP " fma.rn.f32 %7, gu, %16, %7;\n\t"                               \
    "@pt fma.rn.f32 %0, w, %11, %0;\n\t}"

template <bool SAT>
__device__ __forceinline__ void bwd_pixel(float al, float u, float thr, float cutp, float nkap, float ik, float c0,
                                          float c1, float c2, float Gr, float Gg, float Gb, float& T, float& gD,
                                          float& s0, float& s1, float& s2, float& S0, float& S1, float& S2) {
    if (SAT)
        asm(LSB_BWD_BODY("setp.lt.and.f32 pg, %9, 0f3F800000, pt;\n\t", "pg")
            : "+f"(T), "+f"(gD), "+f"(s0), "+f"(s1), "+f"(s2), "+f"(S0), "+f"(S1), "+f"(S2)
            : "f"(thr), "f"(al), "f"(cutp), "f"(nkap), "f"(ik), "f"(c0), "f"(c1), "f"(c2), "f"(u), "f"(0.f),
              "f"(Gr), "f"(Gg), "f"(Gb));
    else
        asm(LSB_BWD_BODY("", "pt")
            : "+f"(T), "+f"(gD), "+f"(s0), "+f"(s1), "+f"(s2), "+f"(S0), "+f"(S1), "+f"(S2)
            : "f"(thr), "f"(al), "f"(cutp), "f"(nkap), "f"(ik), "f"(c0), "f"(c1), "f"(c2), "f"(u), "f"(0.f),
              "f"(Gr), "f"(Gg), "f"(Gb));
}
#undef LSB_BWD_BODY

struct LossArgs {
    const void* observed;    // (H,W,3) f32 or u8 (obs_u8), or NULL: no fused loss
    float* grad;             // (H,W,3) dL/dI out
    double* sums;            // [ntiles*2] tile partials
    double* sums_out;        // [2] totals
    unsigned long long* ticket;    // (unused: the totals come from k_loss_total)
    int kind;                // 0 L1, 1 L2
    float gscale;
    bool obs_u8;             // observed is an 8-bit frame (LSB_OBS_U8)
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Per-warp record pipeline over one tile list [start, end).  `ovr` holds
// one bit per record of the batch being blended: the entry has band pixels
// whose alpha_cut decisions come from the f64 override masks.
struct RecPipe {
    Rec* buf;           // [2][32] in shared memory
    int start, end, slot_next;
    unsigned ovr, ovr_next;
    __device__ __forceinline__ void fetch(const Ws& w, int batch, int slot, int lane) {
        if (slot >= 0) {
            const float4* src = (const float4*)(w.rec + (slot & SLOT_MASK));
            float4* dst = (float4*)(buf + (batch & 1) * 32 + lane);
#pragma unroll
            for (int q = 0; q < 4; ++q) cp_async16(dst + q, src + q);
        }
        cp_commit();
    }
    __device__ __forceinline__ int slot_at(const Ws& w, int j) const { return j < end ? w.tile_slot[j] : -1; }
    // prologue: batch 0 in flight, slots of batch 1 loaded
    __device__ __forceinline__ void begin(const Ws& w, int lane) {
        const int s0 = slot_at(w, start + lane);
        ovr_next = __ballot_sync(0xffffffffu, s0 > 0 && (s0 & OVR_BIT));
        fetch(w, 0, s0, lane);
        slot_next = slot_at(w, start + 32 + lane);
    }
    // start fetching batch b+1, then wait for batch b; returns its records
    __device__ __forceinline__ const Rec* next(const Ws& w, int b, int lane) {
        ovr = ovr_next;
        ovr_next = __ballot_sync(0xffffffffu, slot_next > 0 && (slot_next & OVR_BIT));
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

// Deterministic loss total over the tile partials: one CTA of LT_THREADS;
// thread t adds a contiguous run of tiles in order, then a fixed tree (warp
// butterflies, then the warp sums in order).  Launched after the kernel that
// wrote the partials, so every partial is visible.
constexpr int LT_THREADS = 1024;
__global__ void __launch_bounds__(LT_THREADS) k_loss_total(int ntiles, const double* __restrict__ sums,
                                                         double* __restrict__ out) {
    __shared__ double s0[LT_THREADS / 32], s1[LT_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (ntiles + LT_THREADS - 1) / LT_THREADS;
    double v0 = 0.0, v1 = 0.0;
    for (int j = 0, t = tid * per; j < per && t < ntiles; ++j, ++t) {
        const double2 x = ((const double2*)sums)[t];
        v0 += x.x;
        v1 += x.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    if (lane == 0) {
        s0[warp] = v0;
        s1[warp] = v1;
    }
    __syncthreads();
    if (tid == 0) {
        double a0 = 0.0, a1 = 0.0;
        for (int w = 0; w < LT_THREADS / 32; ++w) {
            a0 += s0[w];
            a1 += s1[w];
        }
        out[0] = a0;
        out[1] = a1;
    }
}

// One record's update of the lane's 8 pixels (rows r0, r0 + 8 of the run)
// in the forward walk.  OVR: the entry has band pixels (per-pixel thresholds
// from the f64 override masks), else the one threshold `cut`.
template <bool COUNT, bool DEPTH, bool OVR>
__device__ __forceinline__ void fwd_pixels(const Frame& f, float4 qb, float4 qc, bool row0, bool row1,
                                           const float* thr, float cut, float nkap, const OvrNib& o,
                                           float (&T)[2][RUN], float (&cnt)[2][RUN], float (&cr)[2][RUN],
                                           float (&cg)[2][RUN], float (&cb)[2][RUN], float (&dz)[2][RUN]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!(h ? row1 : row0)) continue;
        float dy, u0, edy;
        row_terms(f, qb.y, qb.z, 8.f * h, dy, u0, edy);
#pragma unroll
        for (int j = 0; j < RUN; ++j) {
            float u;
            const float al = alpha_sat(qb.x, u0, edy, j, u);
            const float cj = OVR ? ovr_cut(o, h, j, cut) : cut;
            if (!COUNT && !DEPTH)
                fwd_pixel_nc(al, thr[j], cj, nkap, qc.x, qc.y, qc.z, T[h][j], cr[h][j], cg[h][j], cb[h][j]);
            else if (DEPTH)
                fwd_pixel_depth(al, thr[j], cj, nkap, qc.x, qc.y, qc.z, qc.w, T[h][j], cnt[h][j], cr[h][j], cg[h][j],
                                cb[h][j], dz[h][j]);
            else
                fwd_pixel(al, thr[j], cj, nkap, qc.x, qc.y, qc.z, T[h][j], cnt[h][j], cr[h][j], cg[h][j], cb[h][j]);
        }
    }
}

#ifndef LSB_BBOX_FREE
#define LSB_BBOX_FREE 1       // bbox-free records skip the per-pixel bbox test (common.cuh bbox_free_lim)
#endif
#ifndef LSB_FWD_BOTH
#define LSB_FWD_BOTH 1        // fused forward: records reaching both half-tiles walk them without a branch
#endif
#ifndef LSB_PACKED_FWD
#define LSB_PACKED_FWD 1
#endif
// The count-free forward update of one record with packed FP32 (FFMA2 /
// FMUL2 / FADD2 on pixel pairs of the run: half the issue slots of the
// alpha and compositing arithmetic).  Per component the operations are the
// scalar fwd_pixel_nc's (same rounding: mul -> fma multiplicand only, never
// mul -> add, which ptxas would contract for packed operands), and a pair
// that does not composite gets w = 0, so C + 0 c and T + 0 (-clamp) leave
// the accumulators bit-identical to the predicated scalar update.
// w if (T >= thr && a >= cut) else 0: one select on a combined predicate
__device__ __forceinline__ float take_w(float w, float T, float thr, float a, float cut) {
    float r;
    asm("{\n\t.reg .pred p, q;\n\t"
        "setp.ge.f32 p, %2, %3;\n\t"
        "setp.ge.and.f32 q, %4, %5, p;\n\t"
        "selp.f32 %0, %1, 0f00000000, q;\n\t}"
        : "=f"(r)
        : "f"(w), "f"(T), "f"(thr), "f"(a), "f"(cut));
    return r;
}

// BOTH: the caller knows both half-tiles are walked (warp-uniform), so the
// halves carry no branch between them and their pairs can interleave.
template <bool OVR, bool SAT, bool BOTH = false>
__device__ __forceinline__ void fwd_pixels2(const Frame& f, float4 qb, float4 qc, bool row0, bool row1,
                                            const float* thr, float cut, float nkap, const OvrNib& o,
                                            float (&T)[2][RUN], float (&cr)[2][RUN], float (&cg)[2][RUN],
                                            float (&cb)[2][RUN]) {
    const float2 A2 = make_float2(qb.x, qb.x), NK = make_float2(nkap, nkap);
    const float2 C0 = make_float2(qc.x, qc.x), C1 = make_float2(qc.y, qc.y), C2 = make_float2(qc.z, qc.z);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!BOTH && !(h ? row1 : row0)) continue;
        float dy, u0, edy;
        row_terms(f, qb.y, qb.z, 8.f * h, dy, u0, edy);
        const float2 E2 = make_float2(edy, edy), U0 = make_float2(u0, u0);
#pragma unroll
        for (int p = 0; p < RUN / 2; ++p) {
            const int j = 2 * p;
            const float2 u = __fadd2_rn(U0, make_float2((float)j, (float)(j + 1)));
            const float2 q = __ffma2_rn(A2, __fmul2_rn(u, u), E2);
            const float e0 = ex2_approx(q.x), e1 = ex2_approx(q.y);
            const float a0 = SAT ? __saturatef(e0) : e0, a1 = SAT ? __saturatef(e1) : e1;
            float2 t2 = make_float2(T[h][j], T[h][j + 1]);
            float2 w = __fmul2_rn(t2, make_float2(a0, a1));
            const float k0 = OVR ? ovr_cut(o, h, j, cut) : cut, k1 = OVR ? ovr_cut(o, h, j + 1, cut) : cut;
            w.x = take_w(w.x, t2.x, thr[j], a0, k0);
            w.y = take_w(w.y, t2.y, thr[j + 1], a1, k1);
            float2 r2 = __ffma2_rn(w, C0, make_float2(cr[h][j], cr[h][j + 1]));
            float2 g2 = __ffma2_rn(w, C1, make_float2(cg[h][j], cg[h][j + 1]));
            float2 b2 = __ffma2_rn(w, C2, make_float2(cb[h][j], cb[h][j + 1]));
            t2 = __ffma2_rn(w, NK, t2);
            cr[h][j] = r2.x; cr[h][j + 1] = r2.y;
            cg[h][j] = g2.x; cg[h][j + 1] = g2.y;
            cb[h][j] = b2.x; cb[h][j + 1] = b2.y;
            T[h][j] = t2.x; T[h][j + 1] = t2.y;
        }
    }
}

template <bool DEPTH, bool CUT, bool COUNT>
__global__ void __launch_bounds__(32 * WPB, FWD_MIN_BLOCKS)
k_blend_fwd(Ws w, BlendArgs a, LossArgs L, float* __restrict__ image, float* __restrict__ t_final,
            int32_t* __restrict__ n_contrib, float* __restrict__ depth) {
    __shared__ Rec s_rec[WPB][2 * 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int qx = (lane & 3) * RUN, r0 = lane >> 2;      // rows r0 and r0 + 8
    RecPipe pipe;
    pipe.buf = s_rec[wib];
    const float kap = a.clamp;
    // persistent tile-warp: the first tile is the warp's own slot of the
    // heaviest-first order (no atomic), later ones come from the queue,
    // which starts after the first wave.  (Claiming the next slot early, to
    // hide the atomic, costs more in load balance than it saves: +25%.)
    int q0 = blockIdx.x * WPB + wib;
    const int nwarps = gridDim.x * WPB;
    for (;;) {
        int tile = 0;
        if (lane == 0) {
            const int q = q0 >= 0 ? q0 : (int)atomicAdd(&w.ctr[7], 1ull) + nwarps;
            q0 = -1;
            tile = q < w.ntiles ? w.tile_order[q] : -1;
        }
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
        const int gx0 = ox + qx, gy0 = oy + r0;
        const float gx0f = (float)gx0, gy0f = (float)gy0;
        double l0 = 0.0, l1 = 0.0;
        // A pixel composites while T >= t_min (the reference breaks when
        // T < t_min, _kernels.py:98); pixels outside the image start at T = -1.
        float T[2][RUN], cr[2][RUN], cg[2][RUN], cb[2][RUN], dz[2][RUN];
        float cnt[2][RUN];     // processed-entry counts (exact in f32 below 2^24)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                T[h][j] = (gy0 + 8 * h < a.H && gx0 + j < a.W) ? 1.f : -1.f;
                cr[h][j] = cg[h][j] = cb[h][j] = dz[h][j] = 0.f;
                cnt[h][j] = 0.f;
            }
        int last = 0;
        const int start = w.tile_start[tile], end = w.tile_start[tile + 1];
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
                // bbox relative to the lane's run: columns [cx0, cx1), rows [ry0, ry1)
                const int cx0 = (qi.x & 0xffff) - gx0, cx1 = (qi.x >> 16) - gx0;
                const int ry0 = (qi.y & 0xffff) - gy0, ry1 = (qi.y >> 16) - gy0;
                const bool row0 = ry0 <= 0 && ry1 > 0, row1 = ry0 <= 8 && ry1 > 8;
                if (cx0 >= RUN || cx1 <= 0 || !(row0 || row1)) continue;
                if (alive) last = base + k + 1;
                float thr[RUN];                                      // bbox columns of this run
#pragma unroll
                for (int j = 0; j < RUN; ++j) thr[j] = col_thr(j, cx0, cx1, a.tmin);
                const float4 q0 = *(const float4*)&sr[k].mxh;        // mxh myh mxl myl
                const float4 qb = *(const float4*)&sr[k].A;          // A s E lop
                const float4 qc = *(const float4*)&sr[k].kc0;        // clamp * (c0 c1 c2 z)
                const Frame f = frame_of(q0, qb.w, gx0f, gy0f);
                if (CUT && ((pipe.ovr >> k) & 1u))      // band pixels: the f64 decisions
                    fwd_pixels<COUNT, DEPTH, true>(f, qb, qc, row0, row1, thr, a.cutp, -kap,
                                                   ovr_nibbles(w, base + k, lane), T, cnt, cr, cg, cb, dz);
                else
                    fwd_pixels<COUNT, DEPTH, false>(f, qb, qc, row0, row1, thr, CUT ? a.cutp : 0.f, -kap, OvrNib{},
                                                    T, cnt, cr, cg, cb, dz);
            }
            __syncwarp();
        }
        pipe.drain();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        if (lane == 0) w.tile_last[tile] = max(last, start);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gy = gy0 + 8 * h;
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
                if (COUNT) n_contrib[p] = (int32_t)cnt[h][j];
                if (DEPTH) depth[p] = dz[h][j];
                if (L.observed) {
                    const float i3[3] = {ir, ig, ib};
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double d = (double)i3[c] - obs_value(L.observed, L.obs_u8, 3 * p + c);
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
        if (lane == 0) {
            L.sums[2 * tile] = l0;
            L.sums[2 * tile + 1] = l1;
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

// One half-tile (rows r0 + 8h) of the backward for one record: recompute the
// alphas, skip the half when no pixel of it reaches alpha_cut (a superset of
// the exact per-pixel test in bwd_pixel), else update the pixels and fold the
// row sums into the record's moments M.
template <bool SAT, bool OVR = false>
__device__ __forceinline__ void bwd_half(const Frame& f, float4 q1, bool rin, float dyoff, const float* thr,
                                         const BlendArgs& a, float kap, float4 q2, const float* Gr, const float* Gg,
                                         const float* Gb, float* T, float* gD, float* c, float* M,
                                         const OvrNib& o = OvrNib{}, int h = 0) {
    float dy, u0, edy;
    row_terms(f, q1.y, q1.z, dyoff, dy, u0, edy);
    float al[RUN], uu[RUN];
#pragma unroll
    for (int j = 0; j < RUN; ++j) al[j] = alpha_sat<SAT>(q1.x, u0, edy, j, uu[j]);
    if (!OVR) {        // (with band pixels an overridden pair may composite below cut')
        const float amax = fmaxf(fmaxf(al[0], al[1]), fmaxf(al[2], al[3]));
        if (!__any_sync(0xffffffffu, rin && amax >= a.cutp)) return;
    }
    if (!rin) return;
    float S0 = 0.f, S1 = 0.f, S2 = 0.f;
#pragma unroll
    for (int j = 0; j < RUN; ++j)
        bwd_pixel<SAT>(al[j], uu[j], thr[j], OVR ? ovr_cut(o, h, j, a.cutp) : a.cutp, -kap, a.ik, q2.x, q2.y, q2.z,
                       Gr[j], Gg[j], Gb[j], T[j], gD[j], c[0], c[1], c[2], S0, S1, S2);
    M[0] += S0;
    M[1] += S1;
    M[2] = fmaf(S0, dy, M[2]);
    M[3] += S2;
    M[4] = fmaf(S1, dy, M[4]);
    M[5] = fmaf(S0 * dy, dy, M[5]);
}

#ifndef LSB_SMEM_RED
#define LSB_SMEM_RED 1
#endif
// Deferred screen-partial reduction (LSB_SMEM_RED): per record every lane
// parks its 9 raw sums (colour x3, moments x6) in shared memory (3 x 16 B,
// conflict-free), and every RED_RB records the warp reduces them at once:
// lanes 8r..8r+7 own record r of the group, lane sub adds the source lanes
// sub, sub+8, sub+16, sub+24 (LDS.128, one bank group per lane of a
// quarter-warp) and a 3-level butterfly finishes the sum — a fixed tree, so
// deterministic.  The moments -> conic-space map is linear with per-record
// coefficients, so it is applied once to the sums.  Per record this costs
// ~25 warp instructions instead of ~90 for a per-record 9-value
// transpose-reduce.
constexpr int RED_RB = 4;                      // records per deferred reduction
constexpr int RED_F4 = 3;                      // float4 per lane and record

__device__ __forceinline__ void red_park(float4* buf, int slot, int lane, const float* c, const float* M) {
    float4* d = buf + (slot * 32 + lane) * RED_F4;
    d[0] = make_float4(c[0], c[1], c[2], M[0]);
    d[1] = make_float4(M[1], M[2], M[3], M[4]);
    d[2] = make_float4(M[5], 0.f, 0.f, 0.f);
}

// Reduce the `n` parked records (group starting at batch record kb) and
// write their 9 partials per intersection.
__device__ __forceinline__ void red_flush(const Ws& w, const BlendArgs& a, const float4* buf, const Rec* sr, int kb,
                                          int n, int ecur, int lane) {
    __syncwarp();
    const int r = lane >> 3, sub = lane & 7;
    float t[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) t[q] = 0.f;
    if (r < n) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float4* sp = buf + (r * 32 + sub + 8 * j) * RED_F4;
            const float4 x0 = sp[0], x1 = sp[1], x2 = sp[2];
            t[0] += x0.x; t[1] += x0.y; t[2] += x0.z; t[3] += x0.w;
            t[4] += x1.x; t[5] += x1.y; t[6] += x1.z; t[7] += x1.w;
            t[8] += x2.x;
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < 9; ++q) t[q] += __shfl_xor_sync(0xffffffffu, t[q], o);
    const int e = __shfl_sync(0xffffffffu, ecur, kb + (r < n ? r : 0));
    __syncwarp();                                  // the buffer may be refilled from here
    if (r >= n) return;
    const float4 q1 = *(const float4*)&sr[kb + r].A;     // A s E lop
    const float k2 = -2.0f / (float)LOG2E;
    const float ak = q1.x * k2, ek = q1.z * k2, sa = q1.y * ak;
    // moments -> conic-space sums, v0 = a_k u, v1 = s v0 + e dy (all
    // candidates, then a select tree: no divergent branches)
    const float c01 = (sub & 1) ? t[1] : t[0];
    const float c23 = (sub & 1) ? t[3] * (a.ik * ex2_approx(-q1.w)) : t[2];     // 1/op
    const float v45 = (sub & 1) ? fmaf(sa, t[4], ek * t[5]) : ak * t[4];
    const float v67 = 0.5f * ((sub & 1) ? ak * fmaf(sa, t[6], ek * t[7]) : ak * ak * t[6]);
    const float lo = (sub & 2) ? c23 : c01, hi = (sub & 2) ? v67 : v45;
    const float v = (sub & 4) ? hi : (sub < 3 ? lo * a.clamp : lo);
    float* dst = w.part + (int64_t)e * NUM_PART;
    dst[sub] = v;
    if (sub == 0) dst[8] = 0.5f * fmaf(sa * sa, t[6], fmaf(2.f * sa * ek, t[7], ek * ek * t[8]));
}

#ifndef LSB_PACKED_BWD
#define LSB_PACKED_BWD 1
#endif
// The selects of one backward pixel from one predicate pair:
//   take = T >= thr && a >= cut'  -> ws = take ? w : 0
//   gate = take (&& a < 1 with SAT)  -> as = gate ? a : 0
template <bool SAT>
__device__ __forceinline__ void take_wa(float w, float T, float thr, float a, float cut, float& ws, float& as) {
    if (SAT)
        asm("{\n\t.reg .pred p, q, g;\n\t"
            "setp.ge.f32 p, %3, %4;\n\t"
            "setp.ge.and.f32 q, %5, %6, p;\n\t"
            "setp.lt.and.f32 g, %5, 0f3F800000, q;\n\t"
            "selp.f32 %0, %2, 0f00000000, q;\n\t"
            "selp.f32 %1, %5, 0f00000000, g;\n\t}"
            : "=f"(ws), "=f"(as)
            : "f"(w), "f"(T), "f"(thr), "f"(a), "f"(cut));
    else
        asm("{\n\t.reg .pred p, q;\n\t"
            "setp.ge.f32 p, %3, %4;\n\t"
            "setp.ge.and.f32 q, %5, %6, p;\n\t"
            "selp.f32 %0, %2, 0f00000000, q;\n\t"
            "selp.f32 %1, %5, 0f00000000, q;\n\t}"
            : "=f"(ws), "=f"(as)
            : "f"(w), "f"(T), "f"(thr), "f"(a), "f"(cut));
}

// bwd_half with packed FP32 on pixel pairs.  Per component the arithmetic is
// bwd_pixel's (T recurrence bit-identical to the forward's: w = T a, T + ws
// (-clamp) with ws = 0 for a pair that does not composite); the per-record
// sums (colour, moments) are accumulated per pair lane and folded once, and
// the moment sums use fma (S0 + a da, S1 + gd u, S2 + gu u): never a packed
// mul feeding an add, which ptxas would contract.
// The alphas of one half-tile's 4 pixels per lane (2 packed pairs).
template <bool SAT>
__device__ __forceinline__ void bwd_alpha2(const Frame& f, float4 q1, float dyoff, float& dy, float2 (&al)[RUN / 2],
                                           float2 (&uu)[RUN / 2]) {
    float u0, edy;
    row_terms(f, q1.y, q1.z, dyoff, dy, u0, edy);
    const float2 A2 = make_float2(q1.x, q1.x), E2 = make_float2(edy, edy), U0 = make_float2(u0, u0);
#pragma unroll
    for (int p = 0; p < RUN / 2; ++p) {
        uu[p] = __fadd2_rn(U0, make_float2((float)(2 * p), (float)(2 * p + 1)));
        const float2 q = __ffma2_rn(A2, __fmul2_rn(uu[p], uu[p]), E2);
        const float e0 = ex2_approx(q.x), e1 = ex2_approx(q.y);
        al[p] = SAT ? make_float2(__saturatef(e0), __saturatef(e1)) : make_float2(e0, e1);
    }
}

// Per-half sums of the packed backward update (colour x3, moments x3).
struct HalfSums {
    float2 s0, s1, s2, S0, S1, S2;
};

// One packed pixel pair p of a half-tile: the T recurrence bit-identical to
// the forward's (w = T a, T + ws (-clamp) with ws = 0 for a pair that does
// not composite), gD -= w g.c', dL/dalpha, and the pair's terms of the
// record's sums; the moment sums use fma (S0 + a da, S1 + gd u, S2 + gu u):
// never a packed mul feeding an add, which ptxas would contract.
template <bool SAT, bool OVR>
__device__ __forceinline__ void bwd_pair2(int p, float2 al, float2 uu, const float* thr, const BlendArgs& a,
                                          float2 C0, float2 C1, float2 C2, float2 NK, float2 IK, const float* Gr,
                                          const float* Gg, const float* Gb, float* T, float* gD, HalfSums& hs,
                                          const OvrNib& o, int h) {
    const int j = 2 * p;
    float2 t2 = make_float2(T[j], T[j + 1]);
    const float2 w = __fmul2_rn(t2, al);
    float2 ws, as;
    take_wa<SAT>(w.x, t2.x, thr[j], al.x, OVR ? ovr_cut(o, h, j, a.cutp) : a.cutp, ws.x, as.x);
    take_wa<SAT>(w.y, t2.y, thr[j + 1], al.y, OVR ? ovr_cut(o, h, j + 1, a.cutp) : a.cutp, ws.y, as.y);
    const float2 g0 = make_float2(Gr[j], Gr[j + 1]), g1 = make_float2(Gg[j], Gg[j + 1]),
                 g2 = make_float2(Gb[j], Gb[j + 1]);
    const float2 gc = __ffma2_rn(g0, C0, __ffma2_rn(g1, C1, __fmul2_rn(g2, C2)));     // g . c'
    float2 d2 = make_float2(gD[j], gD[j + 1]);
    d2 = __ffma2_rn(make_float2(-ws.x, -ws.y), gc, d2);                             // gD -= w g.c'
    const float2 ia = __fadd2_rn(IK, make_float2(-al.x, -al.y));
    const float2 r = make_float2(rcp_approx(ia.x), rcp_approx(ia.y));
    const float2 da = __ffma2_rn(make_float2(-d2.x, -d2.y), r, __fmul2_rn(t2, gc));  // T g.c' - gD / (1/clamp - a)
    hs.s0 = __ffma2_rn(ws, g0, hs.s0);
    hs.s1 = __ffma2_rn(ws, g1, hs.s1);
    hs.s2 = __ffma2_rn(ws, g2, hs.s2);
    hs.S0 = __ffma2_rn(as, da, hs.S0);                                              // sum gd
    const float2 gd = __fmul2_rn(as, da);
    hs.S1 = __ffma2_rn(gd, uu, hs.S1);                                              // sum gd u
    hs.S2 = __ffma2_rn(__fmul2_rn(gd, uu), uu, hs.S2);                              // sum gd u^2
    t2 = __ffma2_rn(ws, NK, t2);
    T[j] = t2.x;
    T[j + 1] = t2.y;
    gD[j] = d2.x;
    gD[j + 1] = d2.y;
}

__device__ __forceinline__ void half_sums_zero(HalfSums& hs) {
    hs.s0 = make_float2(-0.f, -0.f);
    hs.s1 = hs.s2 = hs.S0 = hs.S1 = hs.S2 = hs.s0;
}

// Fold one half's sums into the record's colour sums c and moments M.
__device__ __forceinline__ void half_sums_fold(const HalfSums& hs, float dy, float* c, float* M) {
    c[0] += hs.s0.x + hs.s0.y;
    c[1] += hs.s1.x + hs.s1.y;
    c[2] += hs.s2.x + hs.s2.y;
    const float m0 = hs.S0.x + hs.S0.y, m1 = hs.S1.x + hs.S1.y, m2 = hs.S2.x + hs.S2.y;
    M[0] += m0;
    M[1] += m1;
    M[2] = fmaf(m0, dy, M[2]);
    M[3] += m2;
    M[4] = fmaf(m1, dy, M[4]);
    M[5] = fmaf(m0 * dy, dy, M[5]);
}

// bwd_half with packed FP32 on pixel pairs (per component bwd_pixel's
// arithmetic; the per-record sums are accumulated per pair lane and folded
// once per half).
template <bool SAT, bool OVR = false>
__device__ __forceinline__ void bwd_half2(const Frame& f, float4 q1, bool rin, float dyoff, const float* thr,
                                          const BlendArgs& a, float kap, float4 q2, const float* Gr, const float* Gg,
                                          const float* Gb, float* T, float* gD, float* c, float* M,
                                          const OvrNib& o = OvrNib{}, int h = 0) {
    float dy;
    float2 al[RUN / 2], uu[RUN / 2];
    bwd_alpha2<SAT>(f, q1, dyoff, dy, al, uu);
    if (!OVR) {        // (with band pixels an overridden pair may composite below cut')
        const float amax = fmaxf(fmaxf(al[0].x, al[0].y), fmaxf(al[1].x, al[1].y));
        if (!__any_sync(0xffffffffu, rin && amax >= a.cutp)) return;
    }
    if (!rin) return;
    const float2 C0 = make_float2(q2.x, q2.x), C1 = make_float2(q2.y, q2.y), C2 = make_float2(q2.z, q2.z);
    const float2 NK = make_float2(-kap, -kap), IK = make_float2(a.ik, a.ik);
    HalfSums hs;
    half_sums_zero(hs);
#pragma unroll
    for (int p = 0; p < RUN / 2; ++p)
        bwd_pair2<SAT, OVR>(p, al[p], uu[p], thr, a, C0, C1, C2, NK, IK, Gr, Gg, Gb, T, gD, hs, o, h);
    half_sums_fold(hs, dy, c, M);
}

// The backward's record walk over one tile's list [start, end): the forward
// recomputed per pixel (same instruction sequence as the forward, so T is
// bit-identical), per-record screen partials reduced across the warp and
// written per intersection; entries the walk never reaches get zeros.
__device__ __forceinline__ void bwd_walk(const Ws& w, const BlendArgs& a, RecPipe& pipe, float4* red, int tile,
                                         int start, int end, int gx0, int gy0, float (&T)[2][RUN],
                                         float (&gD)[2][RUN], float (&Gr)[2][RUN], float (&Gg)[2][RUN],
                                         float (&Gb)[2][RUN], int lane) {
    const float k2 = -2.0f / (float)LOG2E;     // undo the exp2 scaling: a_k = A k2, e = E k2
    const float kap = a.clamp;
    const float gx0f = (float)gx0, gy0f = (float)gy0;
    const int oy = gy0 - (lane >> 2);          // the tile's first row
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
        // intersection ids of this batch, one per lane (written per record below)
        const int ecur = base + lane < end ? w.tile_e[base + lane] : 0;
        const Rec* sr = pipe.next(w, b, lane);
        const int nb = min(32, end - base);
#pragma unroll kBwdUnroll
        for (int k = 0; k < nb; ++k) {
            const float4 q0 = *(const float4*)&sr[k].mxh;        // mxh myh mxl myl
            const float4 q1 = *(const float4*)&sr[k].A;          // A s E lop
            const float4 q2 = *(const float4*)&sr[k].kc0;        // clamp * (c0 c1 c2 z)
            const int4 q3 = *(const int4*)&sr[k].bbx;            // bbx bby id ebase
            // a bbox-free record (warp-uniform, alpha_cut > 0 only): every live
            // lane walks the half-tiles the bbox rows reach, deciding on alpha
            const bool bfree = LSB_BBOX_FREE && a.cut > 0.f && q1.w <= a.bflim;
            bool row0, row1, over;
            int cx0 = 0, cx1 = RUN;
            if (bfree) {
                const int y0 = (q3.y & 0xffff) - oy, y1 = (q3.y >> 16) - oy;
                row0 = y0 < 8 && y1 > 0;
                row1 = y0 < 16 && y1 > 8;
                over = alive;
            } else {
                cx0 = (q3.x & 0xffff) - gx0;
                cx1 = (q3.x >> 16) - gx0;
                const int ry0 = (q3.y & 0xffff) - gy0, ry1 = (q3.y >> 16) - gy0;
                row0 = ry0 <= 0 && ry1 > 0;
                row1 = ry0 <= 8 && ry1 > 8;
                over = alive && cx0 < RUN && cx1 > 0 && (row0 || row1);
            }
            // accumulators: colour (3, x clamp) and the moments sum gd, gd u,
            // gd dy, gd u^2, gd u dy, gd dy^2 with gd = alpha dL/dalpha
            // (-0 is the additive identity the compiler may fold: -0 + x == x for every x)
            float c[3] = {-0.f, -0.f, -0.f}, M[6] = {-0.f, -0.f, -0.f, -0.f, -0.f, -0.f};
            const bool wover = __any_sync(0xffffffffu, over);
            if (wover) {
                // warp-uniform from here: lanes without work get +inf thresholds
                float thr[RUN];
#pragma unroll
                for (int j = 0; j < RUN; ++j)
                    thr[j] = over ? col_thr(j, cx0, cx1, a.tmin) : __int_as_float(0x7f800000);   // (bfree: cx0 0, cx1 RUN)
                const Frame f = frame_of(q0, q1.w, gx0f, gy0f);
#if LSB_PACKED_BWD
#define bwd_half bwd_half2
#endif
                if ((pipe.ovr >> k) & 1u) {            // band pixels: the f64 decisions (saturating form)
                    const OvrNib o = ovr_nibbles(w, base + k, lane);
                    bwd_half<true, true>(f, q1, over && row0, 0.f, thr, a, kap, q2, Gr[0], Gg[0], Gb[0], T[0], gD[0], c,
                                         M, o, 0);
                    bwd_half<true, true>(f, q1, over && row1, 8.f, thr, a, kap, q2, Gr[1], Gg[1], Gb[1], T[1], gD[1], c,
                                         M, o, 1);
                } else if (q1.w >= SAT_LOP) {
                    bwd_half<true>(f, q1, over && row0, 0.f, thr, a, kap, q2, Gr[0], Gg[0], Gb[0], T[0], gD[0], c, M);
                    bwd_half<true>(f, q1, over && row1, 8.f, thr, a, kap, q2, Gr[1], Gg[1], Gb[1], T[1], gD[1], c, M);
                } else {
                    bwd_half<false>(f, q1, over && row0, 0.f, thr, a, kap, q2, Gr[0], Gg[0], Gb[0], T[0], gD[0], c,
                                    M);
                    bwd_half<false>(f, q1, over && row1, 8.f, thr, a, kap, q2, Gr[1], Gg[1], Gb[1], T[1], gD[1], c,
                                    M);
                }
#undef bwd_half
            }
#if LSB_SMEM_RED
            (void)wover;
            red_park(red, k & (RED_RB - 1), lane, c, M);
            if ((k & (RED_RB - 1)) == RED_RB - 1 || k == nb - 1)
                red_flush(w, a, red, sr, k & ~(RED_RB - 1), (k & (RED_RB - 1)) + 1, ecur, lane);
#else
            float val = 0.f;
            if (wover) {
                // moments -> conic-space sums with v0 = a_k u, v1 = s v0 + e dy
                const float ak = q1.x * k2, ek = q1.z * k2, sa = q1.y * ak;
                float v[9];
                v[0] = c[0];
                v[1] = c[1];
                v[2] = c[2];
                v[3] = M[0];
                v[4] = ak * M[1];
                v[5] = fmaf(sa, M[1], ek * M[2]);
                v[6] = ak * ak * M[3];
                v[7] = ak * fmaf(sa, M[3], ek * M[4]);
                v[8] = fmaf(sa * sa, M[3], fmaf(2.f * sa * ek, M[4], ek * ek * M[5]));
                // index i of the 8-vector lands in lanes 4i..4i+3 (reduce8)
                const float r8 = reduce8(v, lane);
                float r9 = v[8];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) r9 += __shfl_xor_sync(0xffffffffu, r9, o);
                val = __shfl_sync(0xffffffffu, r8, 4 * min(lane, 7));
                if (lane == 8) val = r9;
                val *= (lane < 3) ? kap : ((lane == 3) ? a.ik * ex2_approx(-q1.w) : ((lane < 6) ? 1.f : 0.5f));   // 1/op
            }
            const int e = __shfl_sync(0xffffffffu, ecur, k);
            if (lane < NUM_PART) w.part[(int64_t)e * NUM_PART + lane] = val;
#endif
        }
        __syncwarp();
    }
    pipe.drain();
    // intersections the walk never reached contribute nothing
    const int fin = w.tile_start[tile + 1], from = max(end, start);
    for (int z = lane; z < (fin - from) * NUM_PART; z += 32)
        w.part[(int64_t)w.tile_e[from + z / NUM_PART] * NUM_PART + z % NUM_PART] = 0.f;
}

template <bool LOSS>
__global__ void __launch_bounds__(32 * WPB, BWD_MIN_BLOCKS)
k_blend_bwd(Ws w, BlendArgs a, const float* __restrict__ image, const float* __restrict__ gimg, float gscale,
            LossArgs L) {
    __shared__ Rec s_rec[WPB][2 * 32];
    __shared__ float4 s_red[WPB][LSB_SMEM_RED ? RED_RB * 32 * RED_F4 : 1];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int qx = (lane & 3) * RUN, r0 = lane >> 2;
    RecPipe pipe;
    pipe.buf = s_rec[wib];
    // first tile: the warp's own slot of the (heaviest-first) order, no
    // atomic; later tiles from the queue, which starts after the first wave
    int q0 = blockIdx.x * WPB + wib;
    const int nwarps = gridDim.x * WPB;
    for (;;) {
        int tile = 0;
        if (lane == 0) {
            const int q = q0 >= 0 ? q0 : (int)atomicAdd(&w.ctr[8], 1ull) + nwarps;
            q0 = -1;
            tile = q < w.ntiles ? w.tile_order[q] : -1;
        }
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
        const int gx0 = ox + qx, gy0 = oy + r0;
        // per-pixel state: T (as in the forward), gD = g . (I - prefix colour), g = dL/dI
        float T[2][RUN], gD[2][RUN], Gr[2][RUN], Gg[2][RUN], Gb[2][RUN];
        double l0 = 0.0, l1 = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                T[h][j] = -1.f;
                gD[h][j] = Gr[h][j] = Gg[h][j] = Gb[h][j] = 0.f;
                const int gy = gy0 + 8 * h;
                if (gy < a.H && gx0 + j < a.W) {
                    const int64_t p = (int64_t)gy * a.W + gx0 + j;
                    T[h][j] = 1.f;
                    const float i0 = image[3 * p], i1 = image[3 * p + 1], i2 = image[3 * p + 2];
                    float g3[3];
                    if (LOSS) {
                        // photometric loss fused here (optimize.py:48-74, no mask):
                        // dL/dI from (rendered, observed), same arithmetic as the
                        // fused forward / lsb_photometric_loss
                        const float i3[3] = {i0, i1, i2};
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const double d = (double)i3[c] - obs_value(L.observed, L.obs_u8, 3 * p + c);
                            l1 += d * d;
                            if (L.kind == 0) {
                                l0 += fabs(d);
                                g3[c] = d > 0.0 ? L.gscale : (d < 0.0 ? -L.gscale : 0.f);
                            } else {
                                l0 += d * d;
                                g3[c] = (float)(2.0 * d * (double)L.gscale);
                            }
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 3; ++c) g3[c] = gimg[3 * p + c];
                    }
                    Gr[h][j] = g3[0] * gscale;
                    Gg[h][j] = g3[1] * gscale;
                    Gb[h][j] = g3[2] * gscale;
                    gD[h][j] = Gr[h][j] * i0 + Gg[h][j] * i1 + Gb[h][j] * i2;
                }
            }
        if (LOSS) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                l0 += __shfl_xor_sync(0xffffffffu, l0, o);
                l1 += __shfl_xor_sync(0xffffffffu, l1, o);
            }
            if (lane == 0) {
                L.sums[2 * tile] = l0;
                L.sums[2 * tile + 1] = l1;
            }
        }
        bwd_walk(w, a, pipe, s_red[wib], tile, w.tile_start[tile], w.tile_last[tile], gx0, gy0, T, gD, Gr, Gg, Gb,
                 lane);
    }
}

static BlendArgs blend_args(const lsb_settings& s, int W, int H) {
    BlendArgs a{W, H, (float)s.alpha_clamp, (float)s.transmittance_min, (float)s.alpha_cut,
                (float)s.background[0], (float)s.background[1], (float)s.background[2], 0.f, 0.f};
    a.cutp = (float)(s.alpha_cut / s.alpha_clamp);
    a.ik = (float)(1.0 / s.alpha_clamp);
    a.cutlo = (float)(s.alpha_cut / s.alpha_clamp * (1.0 - CUT_BAND));
    a.cuthi = (float)(s.alpha_cut / s.alpha_clamp * (1.0 + CUT_BAND));
    a.clamp_d = s.alpha_clamp;
    a.cut_d = s.alpha_cut;
    a.bflim = bbox_free_lim(s.alpha_cut, s.alpha_clamp, s.footprint_sigma);
    return a;
}

// CTAs to launch for a persistent tile-warp kernel: every resident slot once.
// `reserve` CTA slots per SM are left free for concurrent kernels (the
// window engine's other view lanes: binning and chain co-run with the blend).
static int persistent_grid(const void* fn, int ntiles, int reserve = 0) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * WPB, 0);
    const int need = (ntiles + WPB - 1) / WPB;
    const int g = sms * (per_sm > reserve ? per_sm - reserve : 1);
    return g < need ? g : need;
}

// Forward + photometric loss + backward of one tile in ONE kernel (the window
// engine's step).  Per tile-warp: the count-free forward walk (the same
// instructions as k_blend_fwd<false, CUT, false>), then per pixel the image,
// the loss partials and dL/dI in registers (the same arithmetic as the loss
// fused into k_blend_bwd<true>), then the backward walk over the entries the
// forward reached.  No image, T or gradient image goes through memory, and
// the tile start (queue, ranges, record pipeline) is paid once.
template <bool CUT>
__global__ void __launch_bounds__(32 * WPB, BWD_MIN_BLOCKS)
k_blend_fused(Ws w, BlendArgs a, LossArgs L) {
    __shared__ Rec s_rec[WPB][2 * 32];
    __shared__ float4 s_red[WPB][LSB_SMEM_RED ? RED_RB * 32 * RED_F4 : 1];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int qx = (lane & 3) * RUN, r0 = lane >> 2;
    RecPipe pipe;
    pipe.buf = s_rec[wib];
    const float kap = a.clamp;
    int q0 = blockIdx.x * WPB + wib;
    const int nwarps = gridDim.x * WPB;
    for (;;) {
        int tile = 0;
        if (lane == 0) {
            const int q = q0 >= 0 ? q0 : (int)atomicAdd(&w.ctr[8], 1ull) + nwarps;
            q0 = -1;
            tile = q < w.ntiles ? w.tile_order[q] : -1;
        }
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
        const int gx0 = ox + qx, gy0 = oy + r0;
        const float gx0f = (float)gx0, gy0f = (float)gy0;
        // ---- forward ----
        float T[2][RUN], cr[2][RUN], cg[2][RUN], cb[2][RUN];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                T[h][j] = (gy0 + 8 * h < a.H && gx0 + j < a.W) ? 1.f : -1.f;
                cr[h][j] = cg[h][j] = cb[h][j] = 0.f;
            }
        int last = 0;
        const int start = w.tile_start[tile], end = w.tile_start[tile + 1];
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
#pragma unroll kFusedFwdUnroll
            for (int k = 0; k < nb; ++k) {
                const int4 qi = *(const int4*)&sr[k].bbx;
                const float4 qb = *(const float4*)&sr[k].A;
                bool row0, row1, both = false;
                float thr[RUN];
                if (CUT && LSB_BBOX_FREE && qb.w <= a.bflim) {
                    // bbox-free record (warp-uniform): every pixel decides on alpha alone;
                    // a half-tile is walked iff the bbox rows reach it
                    const int y0 = (qi.y & 0xffff) - oy, y1 = (qi.y >> 16) - oy;
                    row0 = y0 < 8 && y1 > 0;
                    row1 = y0 < 16 && y1 > 8;
                    both = row0 && row1;
#pragma unroll
                    for (int j = 0; j < RUN; ++j) thr[j] = a.tmin;
                } else {
                    const int cx0 = (qi.x & 0xffff) - gx0, cx1 = (qi.x >> 16) - gx0;
                    const int ry0 = (qi.y & 0xffff) - gy0, ry1 = (qi.y >> 16) - gy0;
                    row0 = ry0 <= 0 && ry1 > 0;
                    row1 = ry0 <= 8 && ry1 > 8;
                    if (cx0 >= RUN || cx1 <= 0 || !(row0 || row1)) continue;
#pragma unroll
                    for (int j = 0; j < RUN; ++j) thr[j] = col_thr(j, cx0, cx1, a.tmin);
                }
                if (alive) last = base + k + 1;
                const float4 q0v = *(const float4*)&sr[k].mxh;
                const float4 qc = *(const float4*)&sr[k].kc0;
                const Frame f = frame_of(q0v, qb.w, gx0f, gy0f);
#if LSB_PACKED_FWD
                // (a record with lop < SAT_LOP cannot saturate: its alphas skip the clamp, same bits)
                if (CUT && ((pipe.ovr >> k) & 1u))      // band pixels: the f64 decisions
                    fwd_pixels2<true, true>(f, qb, qc, row0, row1, thr, a.cutp, -kap, ovr_nibbles(w, base + k, lane),
                                            T, cr, cg, cb);
                else if (LSB_FWD_BOTH && CUT && both && qb.w < SAT_LOP)     // the common case: interleaved halves
                    fwd_pixels2<false, false, true>(f, qb, qc, true, true, thr, a.cutp, -kap, OvrNib{}, T, cr, cg,
                                                    cb);
                else if (qb.w >= SAT_LOP)
                    fwd_pixels2<false, true>(f, qb, qc, row0, row1, thr, CUT ? a.cutp : 0.f, -kap, OvrNib{}, T, cr,
                                             cg, cb);
                else
                    fwd_pixels2<false, false>(f, qb, qc, row0, row1, thr, CUT ? a.cutp : 0.f, -kap, OvrNib{}, T, cr,
                                              cg, cb);
#else
                if (CUT && ((pipe.ovr >> k) & 1u))      // band pixels: the f64 decisions
                    fwd_pixels<false, false, true>(f, qb, qc, row0, row1, thr, a.cutp, -kap,
                                                   ovr_nibbles(w, base + k, lane), T, T, cr, cg, cb, T);
                else
                    fwd_pixels<false, false, false>(f, qb, qc, row0, row1, thr, CUT ? a.cutp : 0.f, -kap, OvrNib{},
                                                    T, T, cr, cg, cb, T);
#endif
            }
            __syncwarp();
        }
        pipe.drain();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        last = max(last, start);
        // ---- image, loss, dL/dI ----
        float gD[2][RUN], Gr[2][RUN], Gg[2][RUN], Gb[2][RUN];
        double l0 = 0.0, l1 = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < RUN; ++j) {
                gD[h][j] = Gr[h][j] = Gg[h][j] = Gb[h][j] = 0.f;
                const int gy = gy0 + 8 * h;
                const bool in = gy < a.H && gx0 + j < a.W;
                if (in) {
                    const int64_t p = (int64_t)gy * a.W + gx0 + j;
                    const float i3[3] = {cr[h][j] + T[h][j] * a.bg0, cg[h][j] + T[h][j] * a.bg1,
                                         cb[h][j] + T[h][j] * a.bg2};
                    float g3[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double d = (double)i3[c] - obs_value(L.observed, L.obs_u8, 3 * p + c);
                        l1 += d * d;
                        if (L.kind == 0) {
                            l0 += fabs(d);
                            g3[c] = d > 0.0 ? L.gscale : (d < 0.0 ? -L.gscale : 0.f);
                        } else {
                            l0 += d * d;
                            g3[c] = (float)(2.0 * d * (double)L.gscale);
                        }
                    }
                    Gr[h][j] = g3[0];
                    Gg[h][j] = g3[1];
                    Gb[h][j] = g3[2];
                    gD[h][j] = Gr[h][j] * i3[0] + Gg[h][j] * i3[1] + Gb[h][j] * i3[2];
                }
                T[h][j] = in ? 1.f : -1.f;           // the backward recomputes T from the front
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        if (lane == 0) {
            L.sums[2 * tile] = l0;
            L.sums[2 * tile + 1] = l1;
        }
        // ---- backward ----
        bwd_walk(w, a, pipe, s_red[wib], tile, start, last, gx0, gy0, T, gD, Gr, Gg, Gb, lane);
    }
}

cudaError_t launch_blend_fused(const Ws& w, const lsb_settings& s, int W, int H, const void* observed, int kind,
                               float grad_scale, double* loss_out, cudaStream_t st) {
    const BlendArgs a = blend_args(s, W, H);
    cudaError_t e = cudaMemsetAsync(w.ctr + 8, 0, sizeof(unsigned long long), st);   // tile queue
    if (e != cudaSuccess) return e;
    const LossArgs L{observed, nullptr,     w.loss_part, loss_out,
                     nullptr,  kind & 0xff, grad_scale,  (kind & LSB_OBS_U8) != 0};
    const void* fn = s.alpha_cut > 0.0 ? (const void*)k_blend_fused<true> : (const void*)k_blend_fused<false>;
    const int grid = persistent_grid(fn, w.ntiles, FUSED_RESERVE);
#if LSB_BLEND_PRIO
    // the blend (the step's throughput-limiting kernel) at the device's
    // greatest priority: its CTAs are dispatched ahead of the other lanes'
    // binning / chain CTAs as SM slots free up
    {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(32 * WPB);
        cfg.stream = st;
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributePriority;
        at.val.priority = greatest;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        if (s.alpha_cut > 0.0)
            e = cudaLaunchKernelEx(&cfg, k_blend_fused<true>, w, a, L);
        else
            e = cudaLaunchKernelEx(&cfg, k_blend_fused<false>, w, a, L);
        if (e != cudaSuccess) return e;
    }
#else
    if (s.alpha_cut > 0.0)
        k_blend_fused<true><<<grid, 32 * WPB, 0, st>>>(w, a, L);
    else
        k_blend_fused<false><<<grid, 32 * WPB, 0, st>>>(w, a, L);
#endif
    k_loss_total<<<1, LT_THREADS, 0, st>>>(w.ntiles, w.loss_part, loss_out);
    return cudaGetLastError();
}

static cudaError_t blend_fwd_kernel(const Ws& w, const lsb_settings& s, int W, int H, float* image, float* t_final,
                                    int32_t* n_contrib, float* depth, const void* observed, int kind, float gscale,
                                    float* grad, double* loss_out, cudaStream_t st) {
    const BlendArgs a = blend_args(s, W, H);
    LossArgs L{observed, grad, w.loss_part, loss_out, nullptr, kind & 0xff, gscale, (kind & LSB_OBS_U8) != 0};
    // reset the forward tile queue ([7])
    cudaError_t e = cudaMemsetAsync(w.ctr + 7, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const bool cut = s.alpha_cut > 0.0;
    // n_contrib == NULL (window engine): the count-free forward (no depth)
    if (!n_contrib) {
        const void* fn = cut ? (const void*)k_blend_fwd<false, true, false> : (const void*)k_blend_fwd<false, false, false>;
        const int grid = persistent_grid(fn, w.ntiles);
        if (cut)
            k_blend_fwd<false, true, false><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
        else
            k_blend_fwd<false, false, false><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
        return cudaGetLastError();
    }
    const void* fn = depth ? (cut ? (const void*)k_blend_fwd<true, true, true> : (const void*)k_blend_fwd<true, false, true>)
                           : (cut ? (const void*)k_blend_fwd<false, true, true> : (const void*)k_blend_fwd<false, false, true>);
    const int grid = persistent_grid(fn, w.ntiles);
    if (depth && cut)
        k_blend_fwd<true, true, true><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else if (depth)
        k_blend_fwd<true, false, true><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else if (cut)
        k_blend_fwd<false, true, true><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    else
        k_blend_fwd<false, false, true><<<grid, 32 * WPB, 0, st>>>(w, a, L, image, t_final, n_contrib, depth);
    return cudaGetLastError();
}

cudaError_t launch_blend_fwd(const Ws& w, const lsb_settings& s, int W, int H, float* image, float* t_final,
                             int32_t* n_contrib, float* depth, const void* observed, int kind, float gscale,
                             float* grad, double* loss_out, cudaStream_t st) {
    cudaError_t e = blend_fwd_kernel(w, s, W, H, image, t_final, n_contrib, depth, observed, kind, gscale, grad,
                                     loss_out, st);
    if (e != cudaSuccess || !observed) return e;
    k_loss_total<<<1, LT_THREADS, 0, st>>>(w.ntiles, w.loss_part, loss_out);     // fused loss: the total
    return cudaGetLastError();
}

cudaError_t launch_blend_bwd(const Ws& w, const lsb_settings& s, int W, int H, const float* image,
                             const int32_t* n_contrib, const float* gimg, float gscale, cudaStream_t st) {
    (void)n_contrib;    // liveness is recomputed bit-identically from T
    const BlendArgs a = blend_args(s, W, H);
    cudaError_t e = cudaMemsetAsync(w.ctr + 8, 0, sizeof(unsigned long long), st);   // backward tile queue
    if (e != cudaSuccess) return e;
    const LossArgs L{nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0.f, false};
    k_blend_bwd<false><<<persistent_grid((const void*)k_blend_bwd<false>, w.ntiles), 32 * WPB, 0, st>>>(
        w, a, image, gimg, gscale, L);
    return cudaGetLastError();
}

cudaError_t launch_blend_bwd_loss(const Ws& w, const lsb_settings& s, int W, int H, const float* image,
                                  const void* observed, int kind, float grad_scale, double* loss_out,
                                  cudaStream_t st) {
    const BlendArgs a = blend_args(s, W, H);
    cudaError_t e = cudaMemsetAsync(w.ctr + 8, 0, sizeof(unsigned long long), st);   // backward tile queue
    if (e != cudaSuccess) return e;
    const LossArgs L{observed, nullptr,     w.loss_part, loss_out,
                     nullptr,  kind & 0xff, grad_scale,  (kind & LSB_OBS_U8) != 0};
    k_blend_bwd<true><<<persistent_grid((const void*)k_blend_bwd<true>, w.ntiles), 32 * WPB, 0, st>>>(
        w, a, image, nullptr, 1.0f, L);
    k_loss_total<<<1, LT_THREADS, 0, st>>>(w.ntiles, w.loss_part, loss_out);
    return cudaGetLastError();
}

}  // namespace lsb
