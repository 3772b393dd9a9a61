// Shared device-side definitions for the B200 splat path.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "lsb.h"

namespace lsb {

constexpr int TILE = 16;
constexpr int NUM_PART = 9;          // d_color(3), d_opac, d_mean2d(2), d_cov2d(3)
constexpr int POSE_VALS = 9;         // rho_cam(3), tau_cam(3), d_cam_center(3)
#ifndef LSB_PRE_THREADS
#define LSB_PRE_THREADS 128
#endif
constexpr int PRE_THREADS = LSB_PRE_THREADS;     // preprocess block size
constexpr int PRE_ITEMS = 1;         // Gaussians per preprocess thread
constexpr int CHAIN_BLOCKS = 592;    // fixed grid of the chain kernel (4 x 148 SMs)
constexpr int CHAIN_THREADS = 64;
#ifndef LSB_CHAIN_CH
#define LSB_CHAIN_CH 128
#endif
constexpr int CHAIN_CH = LSB_CHAIN_CH;   // intersections per warp in the chain's partial sums (32 lanes x 4)
constexpr double LOG2E = 1.4426950408889634;

// One visible splat, 64 B, written once by preprocess and read by every tile
// that the splat's bbox touches; the blend copies it to shared memory as is
// (cp.async, 4 x 16 B).  mu_i is kept as an f32 hi/lo pair so a tile can form
// its local coordinate (hi - origin) + lo without f64 arithmetic.  The
// blend works on the saturated alpha a' = min(1, op g / clamp), so the
// record carries log2(op / clamp) and clamp * colour / depth directly.
struct __align__(16) Rec {
    float mxh, myh, mxl, myl;   // mu_i = hi + lo (lo = f32(mu_i - hi))
    float A, s, E, lop;         // log2(op g / clamp) = A*u^2 + E*dy^2 + lop, u = dx + s*dy
    float kc0, kc1, kc2, kz;    // clamp * (clamped RGB), clamp * camera depth (f32 products)
    int32_t bbx, bby;           // x0 | x1 << 16, y0 | y1 << 16 (half-open pixel bbox)
    int32_t id, ebase;          // Gaussian id, first intersection index
};
static_assert(sizeof(Rec) == 64, "Rec must be 64 bytes");

// f64 screen geometry of a visible splat, written by the preprocess whenever
// alpha_cut > 0: mu_i, cov_i (ca, cb, cc), the opacity, and the threshold of
// its alpha >= alpha_cut ellipse d^T cov_i^-1 d <= thr for the
// contributing-list binning mode (lsb_settings.bin_mode = 1; re-read by the
// scatter so both enumerate the same tiles).  The blend re-reads it for the
// rare pairs whose f32 alpha lies within rounding of alpha_cut
// (exact_alpha below).
struct CullGeo {
    double mux, muy, ca, cb, cc, thr, op;
    double c0, c1, c2;            // conic = (cc, -cb, ca) / det, as raster.py:175 forms it
    float kf, sf, ic0f, qcf;      // f32 row form of q for the band search: q = c0 (dx + s dy)^2 + k dy^2,
                                  // 1 / c0, and q at alpha = cut: 2 ln(op / cut)
};
static_assert(sizeof(CullGeo) == 96, "CullGeo is 96 bytes");

// The f64 screen geometry of a visible splat (preprocess, alpha_cut > 0).
__device__ __forceinline__ CullGeo make_cull_geo(double mux, double muy, double ca, double cb, double cc, double thr,
                                                 double op, double cut) {
    CullGeo g;
    g.mux = mux;
    g.muy = muy;
    g.ca = ca;
    g.cb = cb;
    g.cc = cc;
    g.thr = thr;
    g.op = op;
    const double det = __dsub_rn(__dmul_rn(ca, cc), __dmul_rn(cb, cb));
    g.c0 = __ddiv_rn(cc, det);
    g.c1 = __ddiv_rn(-cb, det);
    g.c2 = __ddiv_rn(ca, det);
    const double sr = g.c1 / g.c0;
    g.sf = (float)sr;
    g.kf = (float)(g.c2 - g.c1 * sr);
    g.ic0f = (float)(1.0 / g.c0);
    g.qcf = (float)(2.0 * log(fmax(op / cut, 1e-300)));
    return g;
}

// Relative half-width of the band around alpha_cut inside which the blend's
// f32 alpha (shear-form exponent + ex2.approx) is not trusted to decide
// `alpha < alpha_cut` the way the reference's f64 does: every (pixel, splat)
// pair inside it gets its decision from exact_alpha instead (the tile
// entries that can hold such pairs are flagged before the blend,
// k_band_overrides).  The largest f32 error measured over the band pixels of the
// benchmark views is 1.4e-6 (lsb_render_band_stats), 5.4x inside the band.
#ifndef LSB_CUT_BAND_LOG2
#define LSB_CUT_BAND_LOG2 17
#endif
constexpr double CUT_BAND = 1.0 / (double)(1 << LSB_CUT_BAND_LOG2);
// Bbox-free records.  With alpha_cut > 0 the footprint is nsig =
// min(footprint_sigma, sqrt(2 ln(op / cut))) sigmas (raster.py:160-166).
// When the cut sets it, the bbox square holds the whole ellipse q <= 2 ln(op
// / cut) (its extent along any axis is at most nsig sqrt(lambda_max), the
// bbox radius), i.e. every pixel whose f64 alpha reaches the cut: a pixel
// outside the bbox never composites, so the walks may drop the per-pixel bbox
// test for such a record and decide on alpha alone.  The one exception, f32
// alphas of out-of-bbox pixels inside the alpha_cut band (the sliver just
// beyond the ellipse's extreme points), gets f64 "skip" decisions from the
// band search, which for these records scans the tile, not the bbox.  A
// record is bbox-free iff lop = log2(op / clamp) <= this limit (f32, the same
// value and comparison in the binning and the blend; 0.01 below the exact
// boundary log2(cut / clamp) + fs^2 / (2 ln 2), so lop's rounding cannot
// cross it).
inline float bbox_free_lim(double cut, double clamp, double footprint_sigma) {
    if (!(cut > 0.0)) return -INFINITY;
    return (float)(log2(cut / clamp) + footprint_sigma * footprint_sigma / (2.0 * 0.69314718055994530942) - 0.01);
}

// A sorted tile entry (tile_slot[j]) with band pixels carries this bit; the
// slot is tile_slot[j] & SLOT_MASK.
constexpr int32_t OVR_BIT = 1 << 30;
constexpr int32_t SLOT_MASK = OVR_BIT - 1;

// The reference's alpha in f64 (_kernels.py:64-71): conic = (cc, -cb, ca) /
// det (raster.py:175), q = c0 dx^2 + 2 c1 dx dy + c2 dy^2 left to right
// without contraction, a = min(op exp(-q/2), clamp).  The pair composites
// iff !(a < alpha_cut) (_kernels.py:104).
__device__ __forceinline__ double exact_alpha(const CullGeo& g, double clamp, double px, double py) {
    const double dx = __dsub_rn(px, g.mux), dy = __dsub_rn(py, g.muy);
    double q = __dmul_rn(__dmul_rn(g.c0, dx), dx);
    q = __dadd_rn(q, __dmul_rn(__dmul_rn(__dmul_rn(2.0, g.c1), dx), dy));
    q = __dadd_rn(q, __dmul_rn(__dmul_rn(g.c2, dy), dy));
    const double a = __dmul_rn(g.op, exp(__dmul_rn(-0.5, q)));
    return a > clamp ? clamp : a;
}
struct Ws {
    unsigned long long* ctr;    // [0] M, [1] I, [2] overflow, [3] preprocess ticket, [4] chain ticket,
                                // [5] fused-loss tiles done, [6] big-tile count, [7] fwd / [8] bwd tile queues,
                                // [9] entries flagged OVR_BIT (rows of ovr used), [12] band pixels decided
                                // in f64, [13] of them composited, [14] max relative f32 alpha error there
    Rec* rec;                   // [n] (only the first M are live)
    uint64_t* vkey;             // [n] depth bits of live splats
    uint32_t* colmask;          // [n] interior bits (3) of live splats
    int32_t* tile_count;        // [ntiles]
    int32_t* tile_start;        // [ntiles + 1]
    int32_t* tile_cursor;       // [ntiles]
    int32_t* tile_last;         // [ntiles] one past the last list entry any pixel used
    int32_t* emit_slot;         // [cap] visible slot of intersection e
    int32_t* emit_tile;         // [cap] tile of intersection e
    int32_t* tile_e;            // [cap] intersection index, per-tile depth order
    int32_t* tile_slot;         // [cap] visible slot, per-tile depth order
    int32_t* sort_scratch;      // [cap * 8] fallback sort buffers (tiles > SORT_CAP)
    float* part;                // [cap * NUM_PART] per-intersection gradient partials (AoS)
    int32_t* ovr_of;            // [cap] per intersection e whose entry is flagged OVR_BIT: its row of `ovr`
    uint32_t* ovr;              // [ovr_cap][16]: per flagged (tile, splat) entry, 256-bit masks of the
                                // tile's band pixels [0..7] and of their f64 decisions (1 = composite) [8..15]
    int32_t ovr_cap;
    unsigned long long* sticky; // [1] overflow seen by any render since the caller last cleared it (not
                                // part of the per-render zeroed prefix: lsb_render_sticky reads / clears it)
    double* pose_part;          // [CHAIN_BLOCKS * POSE_VALS]
    double* chain_carry;        // [cap / CHAIN_CH + 1][2][NUM_PART] partial-sum pieces of runs crossing chunks
    double* loss_part;          // [ntiles * 2] fused-loss tile partials
    int32_t* vis_ebase;         // [n + 1] first intersection of each visible slot (exclusive scan)
    int32_t* big_tiles;         // [ntiles] tiles queued for the shared-memory sort
    int32_t* tile_order;        // [ntiles] blend processing order: heaviest tiles first
    CullGeo* cgeo;              // [n] alpha_cut ellipses (bin_mode 1 only)
    uint32_t* warp_mask;        // [ceil(n/32)] visible lanes per preprocess warp
    int32_t* warp_cnt;          // [2 ceil(n/32)] visible count, tile count per warp
    int32_t* warp_off;          // [2 ceil(n/32)] their exclusive scans
    int32_t* chunk_cnt;         // [2 ceil(n/32/1024)] (visible, tile) totals per 1024 preprocess warps
    // the counting pass's full result per visible Gaussian, by Gaussian id
    // (the emitting pass copies it to the Gaussian's slot instead of
    // recomputing the geometry)
    Rec* st_rec;                // [n]
    CullGeo* st_geo;            // [n] (alpha_cut > 0)
    uint64_t* st_key;           // [n]
    uint32_t* st_cm;            // [n]
    int32_t* st_nt;             // [n]
    int64_t n, cap;
    int32_t ntx, nty, ntiles, nblocks_pre;
};

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Carve the caller's workspace; returns the total size needed.
inline size_t carve(const lsb_dims& d, char* base, Ws* w) {
    Ws t{};
    t.n = d.n;
    t.cap = d.isect_cap;
    t.ntx = (d.width + TILE - 1) / TILE;
    t.nty = (d.height + TILE - 1) / TILE;
    t.ntiles = t.ntx * t.nty;
    const int64_t per_block = (int64_t)PRE_THREADS * PRE_ITEMS;
    t.nblocks_pre = (int32_t)((d.n + per_block - 1) / per_block);
    if (t.nblocks_pre < 1) t.nblocks_pre = 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes);
        return base ? (void*)(base + o) : nullptr;
    };
    const size_t n = (size_t)(d.n > 0 ? d.n : 1);
    const size_t cap = (size_t)(d.isect_cap > 0 ? d.isect_cap : 1);
    // first, at a fixed offset whatever the dims (a row band renders through
    // the same workspace with fewer tiles): the sticky overflow flag
    t.sticky = (unsigned long long*)take(sizeof(unsigned long long));
    // zeroed prefix: counters, tile histogram, tile cursors
    t.ctr = (unsigned long long*)take(16 * sizeof(unsigned long long));
    t.tile_count = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.tile_cursor = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.chunk_cnt = (int32_t*)take(sizeof(int32_t) * 2 * (((n + 31) / 32 + 1023) / 1024));
    // not zeroed
    t.tile_start = (int32_t*)take(sizeof(int32_t) * (t.ntiles + 1));
    t.tile_last = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.rec = (Rec*)take(sizeof(Rec) * n);
    t.vkey = (uint64_t*)take(sizeof(uint64_t) * n);
    t.colmask = (uint32_t*)take(sizeof(uint32_t) * n);
    t.emit_slot = (int32_t*)take(sizeof(int32_t) * cap);
    t.emit_tile = (int32_t*)take(sizeof(int32_t) * cap);
    t.tile_e = (int32_t*)take(sizeof(int32_t) * cap);
    t.tile_slot = (int32_t*)take(sizeof(int32_t) * cap);
    t.sort_scratch = (int32_t*)take(sizeof(int32_t) * cap * 8);
    t.part = (float*)take(sizeof(float) * NUM_PART * cap);
    t.ovr_cap = (int32_t)(cap / 16 + 1024);
    t.ovr_of = (int32_t*)take(sizeof(int32_t) * cap);
    t.ovr = (uint32_t*)take(sizeof(uint32_t) * 16 * (size_t)t.ovr_cap);
    t.pose_part = (double*)take(sizeof(double) * CHAIN_BLOCKS * POSE_VALS);
    t.chain_carry = (double*)take(sizeof(double) * 2 * NUM_PART * (cap / CHAIN_CH + 1));
    t.loss_part = (double*)take(sizeof(double) * 2 * t.ntiles);
    t.vis_ebase = (int32_t*)take(sizeof(int32_t) * (n + 1));
    t.big_tiles = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.tile_order = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.cgeo = (CullGeo*)take(sizeof(CullGeo) * n);
    const size_t nw = (n + 31) / 32;
    t.warp_mask = (uint32_t*)take(sizeof(uint32_t) * nw);
    t.warp_cnt = (int32_t*)take(sizeof(int32_t) * 2 * nw);
    t.warp_off = (int32_t*)take(sizeof(int32_t) * 2 * nw);
    t.st_rec = (Rec*)take(sizeof(Rec) * n);
    t.st_geo = (CullGeo*)take(sizeof(CullGeo) * n);
    t.st_key = (uint64_t*)take(sizeof(uint64_t) * n);
    t.st_cm = (uint32_t*)take(sizeof(uint32_t) * n);
    t.st_nt = (int32_t*)take(sizeof(int32_t) * n);
    if (w) *w = t;
    return off;
}

// Bytes of the workspace prefix that must be zeroed before a render
// (counters, tile histograms).
inline size_t zero_prefix_bytes(const Ws& w) {
    return (size_t)((char*)w.tile_start - (char*)w.ctr);
}

// Parameter load from an f32 or f64 arena (lsb_params.dtype), widened to f64.
__device__ __forceinline__ double pld(const void* p, int64_t i, int f64) {
    return f64 ? __ldg((const double*)p + i) : (double)__ldg((const float*)p + i);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---- the blend's f32 alpha (shared with the binning's band search) ---------
constexpr int RUN_PX = 4;    // pixels per lane and row in the blend walks (blend.cu RUN)
// Per-record frame of one lane: the splat mean relative to the lane's first
// pixel (gx0, gy0) and the opacity folded into the exponent.
struct Frame {
    float mxr, myr, lop;
};

__device__ __forceinline__ Frame frame_of(float4 q0, float lop, float gx0f, float gy0f) {
    Frame f;
    f.mxr = __fadd_rn(__fsub_rn(q0.x, gx0f), q0.z);
    f.myr = __fadd_rn(__fsub_rn(q0.y, gy0f), q0.w);
    f.lop = lop;
    return f;
}

// Records with lop below this cannot saturate (a' < 1 for every pixel).
constexpr float SAT_LOP = -1e-6f;

// Row terms: u0 = x_local + s dy - mx at the run's first pixel, and the
// row part of the exponent E dy^2 + log2(op / clamp).
__device__ __forceinline__ void row_terms(const Frame& f, float s, float E, float rowoff, float& dy, float& u0,
                                          float& edy) {
    dy = __fsub_rn(rowoff, f.myr);
    u0 = __fmaf_rn(s, dy, -f.mxr);
    edy = __fmaf_rn(__fmul_rn(E, dy), dy, f.lop);
}

// Saturated alpha of pixel j of the run: a = min(1, op g / clamp).  With
// SAT false the record cannot saturate and the min is dropped.
template <bool SAT = true>
__device__ __forceinline__ float alpha_sat(float A, float u0, float edy, int j, float& u) {
    u = j == 0 ? u0 : __fadd_rn(u0, (float)j);
    const float e = ex2_approx(__fmaf_rn(A, __fmul_rn(u, u), edy));
    return SAT ? __saturatef(e) : e;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Observed camera frames: float32 (H,W,3), or 8-bit (H,W,3) when the loss
// kind carries LSB_OBS_U8 — then the value is u / 255.0 in f64, exactly the
// reference's read_ppm (raster.py:520-541, maxval 255).
// The quotient without a division: q = u * RN(1/255), then one fma residual
// correction, which is the correctly rounded u / 255 for every u in 0..255
// (checked exhaustively on the host: tests/test_frames.py).
__device__ __forceinline__ double u8_unit(unsigned u) {
    const double x = (double)u, r = 1.0 / 255.0;
    const double q = __dmul_rn(x, r);
    return fma(fma(-q, 255.0, x), r, q);
}

__device__ __forceinline__ double obs_value(const void* obs, bool u8, int64_t i) {
    return u8 ? u8_unit(((const uint8_t*)obs)[i]) : (double)((const float*)obs)[i];
}

}  // namespace lsb
