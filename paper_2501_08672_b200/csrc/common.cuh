// Shared device-side definitions for the B200 splat path.
#pragma once
#include <cuda_runtime.h>
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

// Footprint of a splat's alpha >= alpha_cut region for the contributing-list
// binning mode (lsb_settings.bin_mode = 1): the ellipse
// d^T cov_i^-1 d <= thr around mu_i, f64 (written by the preprocess, re-read
// by the scatter so both enumerate the same tiles).
struct CullGeo {
    double mux, muy, ca, cb, cc, thr;
};

struct Ws {
    unsigned long long* ctr;    // [0] M, [1] I, [2] overflow, [3] preprocess ticket, [4] chain ticket,
                                // [5] fused-loss tiles done, [6] big-tile count, [7] fwd / [8] bwd tile queues
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
    double* pose_part;          // [CHAIN_BLOCKS * POSE_VALS]
    double* loss_part;          // [ntiles * 2] fused-loss tile partials
    int32_t* vis_ebase;         // [n + 1] first intersection of each visible slot (exclusive scan)
    int32_t* big_tiles;         // [ntiles] tiles queued for the shared-memory sort
    int32_t* tile_order;        // [ntiles] blend processing order: heaviest tiles first
    CullGeo* cgeo;              // [n] alpha_cut ellipses (bin_mode 1 only)
    uint32_t* warp_mask;        // [ceil(n/32)] visible lanes per preprocess warp
    int32_t* warp_cnt;          // [2 ceil(n/32)] visible count, tile count per warp
    int32_t* warp_off;          // [2 ceil(n/32)] their exclusive scans
    int32_t* chunk_cnt;         // [2 ceil(n/32/1024)] (visible, tile) totals per 1024 preprocess warps
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
    t.pose_part = (double*)take(sizeof(double) * CHAIN_BLOCKS * POSE_VALS);
    t.loss_part = (double*)take(sizeof(double) * 2 * t.ntiles);
    t.vis_ebase = (int32_t*)take(sizeof(int32_t) * (n + 1));
    t.big_tiles = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.tile_order = (int32_t*)take(sizeof(int32_t) * t.ntiles);
    t.cgeo = (CullGeo*)take(sizeof(CullGeo) * n);
    const size_t nw = (n + 31) / 32;
    t.warp_mask = (uint32_t*)take(sizeof(uint32_t) * nw);
    t.warp_cnt = (int32_t*)take(sizeof(int32_t) * 2 * nw);
    t.warp_off = (int32_t*)take(sizeof(int32_t) * 2 * nw);
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
