// K1 preprocess + K2 tile binning (scan, scatter, per-tile depth sort).
//
// This translation unit is compiled with --fmad=false: every f64 operation of
// the projection is rounded exactly where the reference (numpy) rounds it, and
// the one place numpy fuses (the OpenBLAS k=3 dgemm behind `means @ R.T`,
// raster.py:137) is written as explicit __fma_rn.  The discrete decisions —
// near cull, footprint bbox, on-image test, depth order — therefore follow
// the reference's own arithmetic.
#include <cuda_runtime.h>

#include "common.cuh"

#ifndef LSB_SORT_KE
#define LSB_SORT_KE 1       // per-tile warp sort over (depth, e) pairs, slot gathered after
#endif
#ifndef LSB_BAND_SPLAT_MIN_N
#define LSB_BAND_SPLAT_MIN_N 65536   // Gaussians from which the per-splat band search runs
#endif
#ifndef LSB_BAND_SPLAT
#define LSB_BAND_SPLAT 1      // band search per splat (each boundary row once), not per tile entry
#endif

namespace lsb {

struct PreArgs {
    lsb_params p;
    lsb_camera cam;
    lsb_pose T;
    lsb_settings s;
    int degree;
    int cull;          // bin_mode 1 with alpha_cut > 0: contributing tile lists
    int want_geo;      // fill the f64 screen geometry even when alpha_cut == 0 (lsb_splat)
    double* col_out;   // optional: the f64 clipped colour per Gaussian (lsb_splat)
};

// ---- contributing-list binning (bin_mode 1) ---------------------------------
// The blend composites a (pixel, splat) pair only if op g >= alpha_cut, i.e.
// q = d^T cov_i^-1 d <= 2 ln(op / cut) (_kernels.py:104 with the alpha clamp
// folded out).  A tile whose pixels all lie outside that ellipse contributes
// nothing, so mode 1 drops it from the splat's tile set.  The threshold gets a
// margin (0.1% + 0.01) far above the f32 rounding of the blend's own test, so
// no pair the blend would composite is ever dropped: image, T, depth and
// gradients stay bit-identical to the full lists (the dropped entries add
// exact zeros).

__device__ __forceinline__ double cull_thr(double op, double cut) {
    return 2.0 * log(fmax(op / cut, 1.0)) * 1.001 + 0.01;
}

// Pixel columns [c0, c1] of the ellipse over the pixel rows [ya, yb], clipped
// to the bbox columns [x0, x1).  Rows are relaxed to the continuous band
// (a superset); over a band the right edge k dy + w(dy) is concave in dy, so
// its maximum is at the ellipse's rightmost point dy = cb sqrt(thr / ca)
// clamped to the band (mirror for the left edge).
__device__ __forceinline__ bool cull_row_cols(const CullGeo& g, int ya, int yb, int x0, int x1, int& c0, int& c1) {
    const double hy = sqrt(g.thr * g.cc);
    const double da = fmax((double)ya - g.muy, -hy), db = fmin((double)yb - g.muy, hy);
    if (!(da <= db)) return false;
    const double det = g.ca * g.cc - g.cb * g.cb;
    const double k = g.cb / g.cc, w2 = det / g.cc;
    const double dyr = g.cb * sqrt(g.thr / g.ca);
    const double dr = fmin(fmax(dyr, da), db), dl = fmin(fmax(-dyr, da), db);
    const double xr = k * dr + sqrt(fmax(w2 * (g.thr - dr * dr / g.cc), 0.0));
    const double xl = k * dl - sqrt(fmax(w2 * (g.thr - dl * dl / g.cc), 0.0));
    c0 = max(x0, (int)ceil(g.mux + xl));
    c1 = min(x1 - 1, (int)floor(g.mux + xr));
    return c0 <= c1;
}

// Tile range [tx0, tx1] of tile row ty (false if the ellipse misses the row).
__device__ __forceinline__ bool cull_tile_row(const CullGeo& g, int ty, int x0, int x1, int y0, int y1, int& tx0,
                                              int& tx1) {
    int c0, c1;
    if (!cull_row_cols(g, max(ty * TILE, y0), min(ty * TILE + TILE - 1, y1 - 1), x0, x1, c0, c1)) return false;
    tx0 = c0 >> 4;
    tx1 = c1 >> 4;
    return true;
}

__device__ int cull_tile_count(const CullGeo& g, int x0, int x1, int y0, int y1) {
    int n = 0;
    for (int ty = y0 >> 4; ty <= (y1 - 1) >> 4; ++ty) {
        int a, b;
        if (cull_tile_row(g, ty, x0, x1, y0, y1, a, b)) n += b - a + 1;
    }
    return n;
}

__constant__ double c_SH[16] = {
    0.28209479177387814, 0.4886025119029199, 1.0925484305920792, -1.0925484305920792,
    0.31539156525252005, -1.0925484305920792, 0.5462742152960396, -0.5900435899266435,
    2.890611442640554, -0.4570457994644658, 0.3731763325901154, -0.4570457994644658,
    1.445305721320277, -0.5900435899266435, 0.0, 0.0};

// Real SH basis (sh.py:36-63), f64.
__device__ __forceinline__ void sh_basis(int degree, double x, double y, double z, double* b) {
    b[0] = c_SH[0];
    if (degree >= 1) {
        b[1] = -c_SH[1] * y;
        b[2] = c_SH[1] * z;
        b[3] = -c_SH[1] * x;
    }
    if (degree >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[4] = c_SH[2] * x * y;
        b[5] = c_SH[3] * y * z;
        b[6] = c_SH[4] * (2.0 * zz - xx - yy);
        b[7] = c_SH[5] * x * z;
        b[8] = c_SH[6] * (xx - yy);
        if (degree >= 3) {
            b[9] = c_SH[7] * y * (3.0 * xx - yy);
            b[10] = c_SH[8] * x * y * z;
            b[11] = c_SH[9] * y * (4.0 * zz - xx - yy);
            b[12] = c_SH[10] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            b[13] = c_SH[11] * x * (4.0 * zz - xx - yy);
            b[14] = c_SH[12] * z * (xx - yy);
            b[15] = c_SH[13] * x * (xx - 3.0 * yy);
        }
    }
}

// Projection + EWA covariance + footprint (raster.py:134-185) for Gaussian i.
// Returns false if culled; fills the record, its tile count and depth key.
template <bool FULL = true>
__device__ bool splat_one(const PreArgs& a, int64_t i, Rec& r, int& ntiles, uint64_t& key,
                          uint32_t& cmask, CullGeo& geo) {
    const int f64 = a.p.dtype;
    const double px = pld(a.p.means, 3 * i, f64), py = pld(a.p.means, 3 * i + 1, f64),
                 pz = pld(a.p.means, 3 * i + 2, f64);
    const double* R = a.T.R;
    const double* t = a.T.t;
    // mu_c = means @ R^T + t, in the dgemm FMA order
    const double x = __fma_rn(R[2], pz, __fma_rn(R[1], py, R[0] * px)) + t[0];
    const double y = __fma_rn(R[5], pz, __fma_rn(R[4], py, R[3] * px)) + t[1];
    const double z = __fma_rn(R[8], pz, __fma_rn(R[7], py, R[6] * px)) + t[2];
    if (!(z > a.s.near_plane)) return false;
    const double fx = a.cam.fx, fy = a.cam.fy;
    const double mux = fx * x / z + a.cam.cx;
    const double muy = fy * y / z + a.cam.cy;
    // Exact early cull, before the covariance: a splat is kept only with
    // radius <= max_footprint_px =: R, and then x1 <= floor(mux + R) + 1 < 0
    // when mux + R < -1 (x0 >= floor(mux - R) >= W when mux - R >= W; same in
    // y), so its bbox would be empty (raster.py:168-172).
    {
        const double R = a.s.max_footprint_px;
        if (mux + R < -1.0 || mux - R >= (double)a.cam.width || muy + R < -1.0 || muy - R >= (double)a.cam.height)
            return false;
    }
    const double zz = z * z;
    const double J00 = fx / z, J02 = -fx * x / zz;
    const double J11 = fy / z, J12 = -fy * y / zz;
    // world covariance B B^T, B = rot * scale (columns scaled)
    const double s0 = pld(a.p.scales, 3 * i, f64), s1 = pld(a.p.scales, 3 * i + 1, f64),
                 s2 = pld(a.p.scales, 3 * i + 2, f64);
    double B[9];
#pragma unroll
    for (int r3 = 0; r3 < 3; ++r3) {
        B[3 * r3 + 0] = pld(a.p.rots, 9 * i + 3 * r3 + 0, f64) * s0;
        B[3 * r3 + 1] = pld(a.p.rots, 9 * i + 3 * r3 + 1, f64) * s1;
        B[3 * r3 + 2] = pld(a.p.rots, 9 * i + 3 * r3 + 2, f64) * s2;
    }
    // Exact cull with a radius bound, still before the covariance:
    // lambda_max(cov_i) <= |J|_F^2 |B|_F^2 + dilation (spectral <= Frobenius,
    // R_cw orthonormal), and nsig <= footprint_sigma, so the bbox is empty when
    // the centre is farther than that radius (x 1.001 + 1 px against
    // rounding) outside the image.
    {
        double bf = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) bf += B[k] * B[k];
        const double iz = 1.0 / z, xz = x * iz, yz = y * iz;
        const double jf = (fx * iz) * (fx * iz) * (1.0 + xz * xz) + (fy * iz) * (fy * iz) * (1.0 + yz * yz);
        const double rb = a.s.footprint_sigma * sqrt(jf * bf + a.s.dilation) * 1.001 + 1.0;
        if (mux + rb < -1.0 || mux - rb >= (double)a.cam.width || muy + rb < -1.0 || muy - rb >= (double)a.cam.height)
            return false;
    }
    double W[9];
#pragma unroll
    for (int r3 = 0; r3 < 3; ++r3)
#pragma unroll
        for (int c3 = 0; c3 < 3; ++c3)
            W[3 * r3 + c3] = __fma_rn(B[3 * r3 + 2], B[3 * c3 + 2],
                                      __fma_rn(B[3 * r3 + 1], B[3 * c3 + 1], B[3 * r3] * B[3 * c3]));
    // M = J R_cw (2x3)
    double M0[3], M1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        M0[k] = J00 * R[k] + J02 * R[6 + k];
        M1[k] = J11 * R[3 + k] + J12 * R[6 + k];
    }
    // cov_i = M W M^T + dilation I
    double T0[3], T1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T0[k] = M0[0] * W[k] + M0[1] * W[3 + k] + M0[2] * W[6 + k];
        T1[k] = M1[0] * W[k] + M1[1] * W[3 + k] + M1[2] * W[6 + k];
    }
    const double ca = T0[0] * M0[0] + T0[1] * M0[1] + T0[2] * M0[2] + a.s.dilation;
    const double cb = T0[0] * M1[0] + T0[1] * M1[1] + T0[2] * M1[2];
    const double cc = T1[0] * M1[0] + T1[1] * M1[1] + T1[2] * M1[2] + a.s.dilation;
    const double det = ca * cc - cb * cb;
    const double mid = 0.5 * (ca + cc);
    const double amc = ca - cc;
    const double disc = sqrt(fmax(0.25 * (amc * amc) + cb * cb, 0.0));
    const double op = pld(a.p.opacities, i, f64);
    double nsig = a.s.footprint_sigma;
    if (a.s.alpha_cut > 0.0) {
        const double ratio = fmax(op / a.s.alpha_cut, 1.0);
        nsig = fmin(nsig, sqrt(2.0 * log(ratio)));
    }
    const double radius = nsig * sqrt(fmax(mid + disc, 0.0));
    const double W_ = a.cam.width, H_ = a.cam.height;
    const double x0 = fmax(floor(mux - radius), 0.0);
    const double x1 = fmin(floor(mux + radius) + 1.0, W_);
    const double y0 = fmax(floor(muy - radius), 0.0);
    const double y1 = fmin(floor(muy + radius) + 1.0, H_);
    if (!(x0 < x1 && y0 < y1 && radius <= a.s.max_footprint_px)) return false;
    const int ix0 = (int)x0, ix1 = (int)x1, iy0 = (int)y0, iy1 = (int)y1;
    if (a.s.alpha_cut > 0.0 || a.want_geo) geo = make_cull_geo(mux, muy, ca, cb, cc, cull_thr(op, a.s.alpha_cut), op, a.s.alpha_cut);
    if (a.cull) {
        ntiles = cull_tile_count(geo, ix0, ix1, iy0, iy1);
    } else {
        ntiles = (((ix1 - 1) >> 4) - (ix0 >> 4) + 1) * (((iy1 - 1) >> 4) - (iy0 >> 4) + 1);
    }
    if (!FULL) return true;       // counting pass: visibility and tile count only
    // conic = cov_i^-1 = (cc, -cb, ca) / det; exponent in the shear form
    //   q = a_k u^2 + dy^2 / cc,  u = dx - (cb/cc) dy   (no cancellation)
    const double ak = cc / det;
    r.mxh = (float)mux;
    r.myh = (float)muy;
    r.mxl = (float)(mux - (double)r.mxh);
    r.myl = (float)(muy - (double)r.myh);
    r.A = (float)(-0.5 * LOG2E * ak);
    r.s = (float)(-cb / cc);
    r.E = (float)(-0.5 * LOG2E / cc);
    r.lop = (float)(log2(op) - log2(a.s.alpha_clamp));
    // SH colour (raster.py:232-238, sh.py:112-123)
    const double* cc3 = a.T.cam_center;
    const double dvx = px - cc3[0], dvy = py - cc3[1], dvz = pz - cc3[2];
    const double dn = sqrt(dvx * dvx + dvy * dvy + dvz * dvz);
    double dx_ = 0.0, dy_ = 0.0, dz_ = 1.0;
    if (dn > 0.0) {
        const double inv = fmax(dn, 1e-30);
        dx_ = dvx / inv;
        dy_ = dvy / inv;
        dz_ = dvz / inv;
    }
    double b[16];
    sh_basis(a.degree, dx_, dy_, dz_, b);
    const int K = a.p.sh_coeffs;
    const int kk = (a.degree + 1) * (a.degree + 1);
    const int64_t sho = (int64_t)i * K * 3;
    float col[3];
    cmask = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        double acc = b[0] * pld(a.p.shs, sho + c, f64);
#pragma unroll
        for (int k = 1; k < 16; ++k)
            if (k < kk) acc += b[k] * pld(a.p.shs, sho + 3 * k + c, f64);
        const double raw = 0.5 + acc;
        col[c] = (float)fmin(fmax(raw, 0.0), 1.0);
        if (a.col_out) a.col_out[3 * i + c] = fmin(fmax(raw, 0.0), 1.0);
        if (raw > 0.0 && raw < 1.0) cmask |= 1u << c;
    }
    const float kap = (float)a.s.alpha_clamp;
    r.kc0 = __fmul_rn(kap, col[0]);
    r.kc1 = __fmul_rn(kap, col[1]);
    r.kc2 = __fmul_rn(kap, col[2]);
    r.kz = __fmul_rn(kap, (float)z);
    r.bbx = ix0 | (ix1 << 16);
    r.bby = iy0 | (iy1 << 16);
    r.id = (int32_t)i;
    key = (uint64_t)__double_as_longlong(z);
    return true;
}

#ifndef PRE_MIN_BLOCKS
#define PRE_MIN_BLOCKS 1
#endif
// Write a visible splat's record, key and intersections (slot, first
// intersection e0), and bump the tile histogram.
__device__ __forceinline__ void emit_splat(const PreArgs& a, const Ws& w, Rec& r, int64_t slot, int64_t e0, int nt,
                                           uint64_t key, uint32_t cm, const CullGeo& geo) {
    const bool fits = e0 + nt <= w.cap;
    r.ebase = fits ? (int32_t)e0 : -1;
    w.rec[slot] = r;
    w.vis_ebase[slot] = (int32_t)min(e0, (int64_t)0x7fffffff);
    w.vkey[slot] = key;
    w.colmask[slot] = cm;
    if (a.s.alpha_cut > 0.0) w.cgeo[slot] = geo;     // the blend's f64 alpha_cut decisions (exact_alpha)
    if (!fits) return;
    const int x0 = r.bbx & 0xffff, x1 = r.bbx >> 16, y0 = r.bby & 0xffff, y1 = r.bby >> 16;
    // tile histogram, and each intersection's (slot, tile) for the scatter,
    // e running row-major over the splat's tiles from e0
    int e = (int)e0;
    if (a.cull) {
        for (int ty = y0 >> 4; ty <= (y1 - 1) >> 4; ++ty) {
            int tx0, tx1;
            if (!cull_tile_row(geo, ty, x0, x1, y0, y1, tx0, tx1)) continue;
            for (int tx = tx0; tx <= tx1; ++tx, ++e) {
                atomicAdd(&w.tile_count[ty * w.ntx + tx], 1);
                w.emit_tile[e] = ty * w.ntx + tx;
                w.emit_slot[e] = (int32_t)slot;
                if (LSB_BAND_SPLAT) w.ovr_of[e] = -1;
            }
        }
        return;
    }
    for (int ty = y0 >> 4; ty <= (y1 - 1) >> 4; ++ty)
        for (int tx = x0 >> 4; tx <= (x1 - 1) >> 4; ++tx, ++e) {
            atomicAdd(&w.tile_count[ty * w.ntx + tx], 1);
            w.emit_tile[e] = ty * w.ntx + tx;
            w.emit_slot[e] = (int32_t)slot;
            if (LSB_BAND_SPLAT) w.ovr_of[e] = -1;
        }
}

// Exclusive scan of the tile histogram (single CTA: the counts are staged in
// shared memory once; each thread owns a run of consecutive tiles), then the
// heaviest-first processing order of the tiles.
constexpr int ST_THREADS = 1024;
__global__ void __launch_bounds__(ST_THREADS) k_scan_tiles(Ws w) {
    __shared__ int s_w[ST_THREADS / 32];
    // the tile counts, staged once (coalesced); skewed by one word per 32 so
    // the per-thread runs below read distinct banks
    extern __shared__ int s_cnt[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (w.ctr[1] > (unsigned long long)w.cap) {
        // capacity overflow: splats past the capacity emitted nothing, so the
        // intersection arrays are incomplete — publish empty tiles (nothing
        // downstream reads them) and let the caller regrow and retry
        for (int i = tid; i <= w.ntiles; i += ST_THREADS) w.tile_start[i] = 0;
        for (int i = tid; i < w.ntiles; i += ST_THREADS) w.tile_order[i] = i;
        return;
    }
    for (int i = tid; i < w.ntiles; i += ST_THREADS) s_cnt[i + (i >> 5)] = w.tile_count[i];
    __syncthreads();
    const int per = (w.ntiles + ST_THREADS - 1) / ST_THREADS;
    const int b0 = tid * per;
    int sum = 0;
    for (int i = 0; i < per; ++i)
        if (b0 + i < w.ntiles) sum += s_cnt[b0 + i + ((b0 + i) >> 5)];
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {                     // exclusive scan of the warp totals
        const int tv = s_w[lane];
        int z = tv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        s_w[lane] = z - tv;
    }
    __syncthreads();
    int run = x - sum + s_w[warp];
    for (int i = 0; i < per; ++i)
        if (b0 + i < w.ntiles) {
            w.tile_start[b0 + i] = run;
            run += s_cnt[b0 + i + ((b0 + i) >> 5)];
        }
    if (tid == ST_THREADS - 1) w.tile_start[w.ntiles] = run;
    // Processing order of the persistent blend kernels: a counting sort of
    // the tiles by descending list length (4-entry buckets), so the longest
    // tiles start first and the tail of the tile queue is short work.
    // (warp-aggregated: most tiles share a few buckets, and same-address
    // shared atomics serialise)
    __shared__ int s_hist[256];
    if (tid < 256) s_hist[tid] = 0;
    __syncthreads();
    auto key = [](int c) { return 255 - min(c >> 2, 255); };
    for (int i = 0; i < per; ++i) {
        const bool ok = b0 + i < w.ntiles;
        const int k = ok ? key(s_cnt[b0 + i + ((b0 + i) >> 5)]) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, k);
        if (ok && lane == __ffs(grp) - 1) atomicAdd(&s_hist[k], __popc(grp));
    }
    __syncthreads();
    if (warp == 0) {
        int loc[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            loc[i] = tot;
            tot += s_hist[8 * lane + i];
        }
        int y = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int z = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += z;
        }
        const int excl = y - tot;
#pragma unroll
        for (int i = 0; i < 8; ++i) s_hist[8 * lane + i] = excl + loc[i];
    }
    __syncthreads();
    for (int i = 0; i < per; ++i) {
        const bool ok = b0 + i < w.ntiles;
        const int k = ok ? key(s_cnt[b0 + i + ((b0 + i) >> 5)]) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, k);
        const int leader = __ffs(grp) - 1;
        int base = 0;
        if (ok && lane == leader) base = atomicAdd(&s_hist[k], __popc(grp));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (ok) w.tile_order[base + __popc(grp & ((1u << lane) - 1u))] = b0 + i;
    }
}

// sqrt(x) for x >= 0 from the MUFU reciprocal square root (the band search
// widens its annulus far beyond this rounding).
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return x > 0.f ? x * r : 0.f;
}

// The alpha_cut band of one (splat, tile) entry.  The blend decides `alpha <
// alpha_cut` (_kernels.py:104) in f32; where its f32 alpha may lie too close
// to the cut for that to be the reference's f64 decision, the entry carries
// OVR_BIT and a row of 256-bit masks (the band pixels of the tile and their
// decisions taken here in f64 with exact_alpha), which the blend follows.
// The search: the pixel centres of the tile (inside the splat's bbox) in the
// annulus |q - qc| <= W around q = qc = 2 ln(op / cut), row by row from the
// roots of the row's quadratic q = c0 (dx + s dy)^2 + k dy^2 (f32, tile-
// relative centre from f64).  W covers 2 CUT_BAND plus this search's own f32
// error, so every pixel whose alpha / cut lies within 1 +- CUT_BAND is found;
// the blend's f32 alpha is at least 5x more accurate than CUT_BAND.  For each
// band pixel the f32 alpha the blend computes (same instruction sequence and
// lane frame) is also formed and the largest relative error against the f64
// one is kept in ctr[14] (the evidence for the band width).  Nearly every
// entry has no band pixel and costs a few instructions per tile row.
// One band pixel (tile-relative x, ry) of an entry: allocate the entry's
// mask row at its first band pixel (idx < 0), take the f64 decision, record
// it, and keep the f32-error evidence.  Returns the row, or -1 when the mask
// table is full (reported as a capacity overflow: regrow and redo).
__device__ __forceinline__ int band_pixel(const Ws& w, const CullGeo& g, const Rec& r, double clamp, double cut, int idx,
                                       int ox, int oy, int x, int ry, bool inbox) {
    if (idx < 0) {
        idx = (int)atomicAdd(&w.ctr[9], 1ull);
        if (idx >= w.ovr_cap) {
            w.ctr[2] = 1;
            *w.sticky = 1ull;
            return -1;
        }
        for (int q = 0; q < 16; ++q) w.ovr[(size_t)idx * 16 + q] = 0u;
    }
    const double ad = exact_alpha(g, clamp, (double)(ox + x), (double)(oy + ry));
    const bool take = inbox && !(ad < cut);       // outside the bbox: not in the pixel's list
    const int bit = ry * TILE + x;
    uint32_t* m = w.ovr + (size_t)idx * 16;
    m[bit >> 5] |= 1u << (bit & 31);
    if (take) m[8 + (bit >> 5)] |= 1u << (bit & 31);
    atomicAdd(&w.ctr[12], 1ull);
    if (take) atomicAdd(&w.ctr[13], 1ull);
    // the blend's own f32 alpha for this pixel (its lane's frame)
    const Frame f = frame_of(*(const float4*)&r.mxh, r.lop, (float)(ox + (x & ~(RUN_PX - 1))), (float)(oy + (ry & 7)));
    float dyf, u0, edy, u;
    row_terms(f, r.s, r.E, 8.f * (float)(ry >> 3), dyf, u0, edy);
    const float al = alpha_sat(r.A, u0, edy, x & (RUN_PX - 1), u);
    atomicMax((unsigned int*)&w.ctr[14], __float_as_uint((float)fabs((double)al * clamp / ad - 1.0)));
    return idx;
}

__device__ __forceinline__ bool band_search(const Ws& w, double clamp, double cut, float bflim, int64_t e, int slot,
                                            int tile) {
    const CullGeo& g = w.cgeo[slot];
    const float qc = g.qcf;
    const float W = (float)(4.0 * CUT_BAND) + 4e-6f * fabsf(qc) + 1e-6f;
    const float qo = qc + W, qi = qc - W;
    if (qo < 0.f) return false;              // op below the band: no pair comes near the cut
    const int ox = (tile % w.ntx) * TILE, oy = (tile / w.ntx) * TILE;
    const Rec& r = w.rec[slot];
    const int x0 = r.bbx & 0xffff, x1 = r.bbx >> 16, y0 = r.bby & 0xffff, y1 = r.bby >> 16;
    const float mxr = (float)(g.mux - (double)ox), myr = (float)(g.muy - (double)oy);
    const float k = g.kf, sr = g.sf, ic0 = g.ic0f;
    // a bbox-free record (bbox_free_lim) is searched over the whole tile, not
    // only its bbox: out-of-bbox band pixels get "skip"
    const bool bf = r.lop <= bflim;
    const int bx0 = bf ? ox : x0, bx1 = bf ? ox + TILE : x1, by0 = bf ? oy : y0, by1 = bf ? oy + TILE : y1;
    const int cx0 = max(ox, bx0) - ox, cx1 = min(ox + TILE, bx1) - 1 - ox;     // tile-relative columns
    const float dyx = sqrt_approx(qo / k) + 1e-3f;
    const int ry0 = max(max(0, by0 - oy), __float2int_ru(myr - dyx));
    const int ry1 = min(min(TILE, by1 - oy), __float2int_rd(myr + dyx) + 1);
    if (ry0 >= ry1 || cx0 > cx1) return false;
    // an entry whose pixel rectangle lies inside the inner ellipse has no band
    // pixel: q is convex, so its maximum over the rectangle is at a corner
    {
        const float c0 = (float)g.c0;
        const float da = (float)ry0 - myr, db = (float)(ry1 - 1) - myr;
        const float ua = __fmaf_rn(sr, da, (float)cx0 - mxr), ub = __fmaf_rn(sr, db, (float)cx0 - mxr);
        const float w = (float)(cx1 - cx0);
        const float va = k * da * da, vb = k * db * db;
        const float qmax = fmaxf(fmaxf(__fmaf_rn(c0 * ua, ua, va), __fmaf_rn(c0 * (ua + w), ua + w, va)),
                                 fmaxf(__fmaf_rn(c0 * ub, ub, vb), __fmaf_rn(c0 * (ub + w), ub + w, vb)));
        if (qmax < qi * 0.999f) return false;
    }
    int idx = -1;
    for (int ry = ry0; ry < ry1; ++ry) {
        const float dy = (float)ry - myr;
        const float v = k * dy * dy;
        const float to = qo - v;
        if (to < 0.f) continue;
        const float xm = __fmaf_rn(-sr, dy, mxr);        // the row's centre
        const float ho = sqrt_approx(to * ic0);
        const int xa = max(cx0, __float2int_ru(xm - ho));
        const int xb = min(cx1, __float2int_rd(xm + ho));
        if (xa > xb) continue;
        const float ti = qi - v;
        const float hi = ti > 0.f ? sqrt_approx(ti * ic0) : -1.f;
        // candidates |x - xm| >= hi: the left run up to xm - hi, the right run from xm + hi
        const int xl = hi < 0.f ? xb : __float2int_rd(xm - hi);
        const int xr = hi < 0.f ? xb + 1 : __float2int_ru(xm + hi);
        if (xl < xa && xr > xb) continue;                 // the segment lies inside the inner ellipse
        for (int x = xa; x <= xb; ++x) {
            if (x > xl && x < xr) x = xr;                 // jump over the inner run
            if (x > xb) break;
            const bool inbox = ox + x >= x0 && ox + x < x1 && oy + ry >= y0 && oy + ry < y1;
            idx = band_pixel(w, g, r, clamp, cut, idx, ox, oy, x, ry, inbox);
            if (idx < 0) return false;                    // (no room: a capacity overflow was reported)
        }
    }
    if (idx < 0) return false;
    w.ovr_of[e] = idx;
    return true;
}

#ifndef LSB_BAND_GROUP
#define LSB_BAND_GROUP 2     // (measured: 1, 2, 4, 8, 16, 32 lanes; 2 the fastest)
#endif
constexpr int BAND_GROUP = LSB_BAND_GROUP;     // lanes per splat in k_band_splats

// The alpha_cut band of every visible splat at once: the same annulus
// |q - qc| <= W as band_search, walked once per pixel row of the splat's
// search region (its bbox; for a bbox-free record the tile hull of the bbox)
// instead of once per row of every tile entry, BAND_GROUP lanes per splat
// taking its rows in turn.  A candidate pixel joins the entry of its tile
// (if the splat emitted that tile): band_pixel, with ovr_of[e] (-1 from the
// emitting pass) holding the entry's mask row.  Candidates are rare, so the
// lanes holding some take them one lane at a time (entries are never
// shared between two lanes' band_pixel calls at once).
__global__ void __launch_bounds__(256) k_band_splats(Ws w, double clamp, double cut, float bflim) {
    if (w.ctr[1] > (unsigned long long)w.cap) return;     // overflow: tiles published empty
    const int64_t M = (int64_t)w.ctr[0];
    const int lane = threadIdx.x & 31, sub = lane & (BAND_GROUP - 1);
    const int64_t groups = (int64_t)gridDim.x * (blockDim.x / BAND_GROUP);
    const int64_t g0 = (int64_t)blockIdx.x * (blockDim.x / BAND_GROUP) + (threadIdx.x / BAND_GROUP);
    // warp-uniform trip count over the slots
    const int64_t wbase = g0 - (lane / BAND_GROUP);
    for (int64_t sb = wbase; sb < M; sb += groups) {
        const int64_t slot = sb + lane / BAND_GROUP;
        const bool live = slot < M;
        float qo = -1.f, qi = 0.f, mxr = 0.f, myr = 0.f, k = 0.f, sr = 0.f, ic0 = 0.f;
        int ox = 0, oy = 0, cx0 = 0, cx1 = -1, ry0 = 0, ry1 = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
        bool bf = false;
        if (live) {
            const CullGeo& g = w.cgeo[slot];
            const float qc = g.qcf;
            const float W = (float)(4.0 * CUT_BAND) + 4e-6f * fabsf(qc) + 1e-6f;
            qo = qc + W;
            qi = qc - W;
            const Rec& r = w.rec[slot];
            x0 = r.bbx & 0xffff; x1 = r.bbx >> 16; y0 = r.bby & 0xffff; y1 = r.bby >> 16;
            bf = r.lop <= bflim;
            ox = x0 & ~(TILE - 1);
            oy = y0 & ~(TILE - 1);
            const int bx1 = bf ? (((x1 - 1) | (TILE - 1)) + 1) : x1, by1 = bf ? (((y1 - 1) | (TILE - 1)) + 1) : y1;
            const int bx0 = bf ? ox : x0, by0 = bf ? oy : y0;
            mxr = (float)(g.mux - (double)ox);
            myr = (float)(g.muy - (double)oy);
            k = g.kf; sr = g.sf; ic0 = g.ic0f;
            cx0 = bx0 - ox;
            cx1 = bx1 - 1 - ox;
            if (qo >= 0.f) {
                const float dyx = sqrt_approx(qo / k) + 1e-3f;
                ry0 = max(by0 - oy, __float2int_ru(myr - dyx));
                ry1 = min(by1 - oy, __float2int_rd(myr + dyx) + 1);
            }
        }
        int rounds = ry1 > ry0 ? (ry1 - ry0 + BAND_GROUP - 1) / BAND_GROUP : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
        for (int j = 0; j < rounds; ++j) {
            const int ry = ry0 + j * BAND_GROUP + sub;
            int xa = 0, xb = -1, xl = 0, xr = 0;
            bool has = false;
            if (ry < ry1) {
                const float dy = (float)ry - myr;
                const float v = k * dy * dy;
                const float to = qo - v;
                if (to >= 0.f) {
                    const float xm = __fmaf_rn(-sr, dy, mxr);
                    const float ho = sqrt_approx(to * ic0);
                    xa = max(cx0, __float2int_ru(xm - ho));
                    xb = min(cx1, __float2int_rd(xm + ho));
                    const float ti = qi - v;
                    const float hi = ti > 0.f ? sqrt_approx(ti * ic0) : -1.f;
                    xl = hi < 0.f ? xb : __float2int_rd(xm - hi);
                    xr = hi < 0.f ? xb + 1 : __float2int_ru(xm + hi);
                    has = xa <= xb && !(xl < xa && xr > xb);
                }
            }
            unsigned pend = __ballot_sync(0xffffffffu, has);
            while (pend) {
                const int src = __ffs(pend) - 1;
                pend &= pend - 1;
                if (lane == src) {
                    const CullGeo& g = w.cgeo[slot];
                    const Rec& r = w.rec[slot];
                    const int e0 = w.vis_ebase[slot], e1 = w.vis_ebase[slot + 1];
                    for (int x = xa; x <= xb; ++x) {
                        if (x > xl && x < xr) x = xr;             // jump over the inner run
                        if (x > xb) break;
                        const int X = ox + x, Y = oy + ry;
                        const bool inbox = X >= x0 && X < x1 && Y >= y0 && Y < y1;
                        const int t = (Y >> 4) * w.ntx + (X >> 4);
                        int e = -1;
                        for (int q = e0; q < e1; ++q)
                            if (w.emit_tile[q] == t) { e = q; break; }
                        if (e < 0) continue;                        // a tile the splat did not emit
                        const int idx = w.ovr_of[e];
                        const int nidx = band_pixel(w, g, r, clamp, cut, idx, X & ~(TILE - 1), Y & ~(TILE - 1),
                                                    X & (TILE - 1), Y & (TILE - 1), inbox);
                        if (nidx < 0) break;                        // (no room: a capacity overflow was reported)
                        if (idx < 0) w.ovr_of[e] = nidx;
                    }
                }
                __syncwarp();
            }
        }
    }
}

// Scatter with the (slot, tile) pairs the preprocess emitted: one thread per
// intersection claims a position in its tile's bucket (and, with alpha_cut
// > 0, searches its entry for alpha_cut band pixels: band_search).
__global__ void __launch_bounds__(256) k_scatter_emitted(Ws w, double clamp, double cut, float bflim, int splat_band) {
    if (w.ctr[1] > (unsigned long long)w.cap) return;     // overflow: tiles published empty
    const int64_t I = (int64_t)w.ctr[1];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < I; e += stride) {
        const int t = w.emit_tile[e];
        const int slot = w.emit_slot[e];
        const int j = w.tile_start[t] + atomicAdd(&w.tile_cursor[t], 1);
        // splat_band: k_band_splats already searched (band pixels found in
        // the entry: ovr_of[e] >= 0); else the entry is searched here
        const bool band = cut > 0.0 && (splat_band ? w.ovr_of[e] >= 0 : band_search(w, clamp, cut, bflim, e, slot, t));
        w.tile_e[j] = (int32_t)e;
        w.tile_slot[j] = slot | (band ? OVR_BIT : 0);      // the flag rides on the slot (sorts mask it)
    }
}

constexpr int SORT_CAP = 4096;   // entries sorted entirely in shared memory

// (slots may carry OVR_BIT: compared and indexed without it)
__device__ __forceinline__ bool key_less(uint64_t ka, int sa, uint64_t kb, int sb) {
    sa &= SLOT_MASK;
    sb &= SLOT_MASK;
    return ka < kb || (ka == kb && sa < sb);
}

// Bitonic sort of n <= SORT_CAP (depth, slot) keys held in shared memory.
__device__ void smem_bitonic(uint64_t* k, int* s, int* e, int n) {
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = n + threadIdx.x; i < P; i += blockDim.x) {
        k[i] = ~0ull;
        s[i] = 0x7fffffff;
        e[i] = -1;
    }
    __syncthreads();
    for (int kk = 2; kk <= P; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & kk) == 0;
                    const bool lt = key_less(k[ixj], s[ixj], k[i], s[i]);
                    if (lt == up) {
                        const uint64_t tk = k[i]; k[i] = k[ixj]; k[ixj] = tk;
                        const int ts = s[i]; s[i] = s[ixj]; s[ixj] = ts;
                        const int te = e[i]; e[i] = e[ixj]; e[ixj] = te;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Bitonic sort of up to 32*R (depth, slot, e) triples held in registers by
// one warp: element i lives in lane (i & 31), register (i >> 5).
template <int R>
__device__ void warp_bitonic(uint64_t* k, int* s, int* e, int lane) {
    constexpr int P = 32 * R;
#pragma unroll
    for (int kk = 2; kk <= P; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int rp = r ^ jr;
                    if (rp > r) {
                        const int i = r * 32 + lane;
                        const bool up = (i & kk) == 0;
                        const bool lt = key_less(k[rp], s[rp], k[r], s[r]);
                        if (lt == up) {
                            const uint64_t tk = k[r]; k[r] = k[rp]; k[rp] = tk;
                            const int ts = s[r]; s[r] = s[rp]; s[rp] = ts;
                            const int te = e[r]; e[r] = e[rp]; e[rp] = te;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = r * 32 + lane;
                    const uint64_t ok = __shfl_xor_sync(0xffffffffu, k[r], j);
                    const int os = __shfl_xor_sync(0xffffffffu, s[r], j);
                    const int oe = __shfl_xor_sync(0xffffffffu, e[r], j);
                    const bool up = (i & kk) == 0;
                    const bool lower = (lane & j) == 0;
                    // lower element keeps the smaller key when ascending
                    const bool other_less = key_less(ok, os, k[r], s[r]);
                    const bool take = (lower == up) ? other_less : !other_less;
                    if (take) { k[r] = ok; s[r] = os; e[r] = oe; }
                }
            }
        }
    }
}

// warp_bitonic over (depth, x) pairs, x = e with OVR_BIT (compared without it).
template <int R>
__device__ void warp_bitonic_ke(uint64_t* k, int* x, int lane) {
    constexpr int P = 32 * R;
#pragma unroll
    for (int kk = 2; kk <= P; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int rp = r ^ jr;
                    if (rp > r) {
                        const int i = r * 32 + lane;
                        const bool up = (i & kk) == 0;
                        const bool lt = key_less(k[rp], x[rp], k[r], x[r]);
                        if (lt == up) {
                            const uint64_t tk = k[r]; k[r] = k[rp]; k[rp] = tk;
                            const int tx = x[r]; x[r] = x[rp]; x[rp] = tx;
                        }
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = r * 32 + lane;
                    const uint64_t ok = __shfl_xor_sync(0xffffffffu, k[r], j);
                    const int ox = __shfl_xor_sync(0xffffffffu, x[r], j);
                    const bool up = (i & kk) == 0;
                    const bool lower = (lane & j) == 0;
                    const bool other_less = key_less(ok, ox, k[r], x[r]);
                    const bool take = (lower == up) ? other_less : !other_less;
                    if (take) { k[r] = ok; x[r] = ox; }
                }
            }
        }
    }
}

template <int R>
__device__ void warp_sort_tile(const Ws& w, int start, int n, int lane) {
    uint64_t k[R];
    int s[R], e[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = r * 32 + lane;
        if (i < n) {
            e[r] = w.tile_e[start + i];
            s[r] = w.tile_slot[start + i];
            k[r] = w.vkey[s[r] & SLOT_MASK];
        } else {
            k[r] = ~0ull;
            s[r] = 0x7fffffff;
            e[r] = -1;
        }
    }
#if LSB_SORT_KE
    // (depth, e) pairs: a tile holds one entry per splat and e runs in slot
    // order (vis_ebase), so e breaks depth ties exactly as the slot does; the
    // slot (with the entry's OVR_BIT, carried on e) is gathered after the sort
#pragma unroll
    for (int r = 0; r < R; ++r) e[r] = (r * 32 + lane < n) ? (e[r] | (s[r] & OVR_BIT)) : SLOT_MASK;
    warp_bitonic_ke<R>(k, e, lane);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = r * 32 + lane;
        if (i < n) {
            const int ee = e[r] & SLOT_MASK;
            w.tile_e[start + i] = ee;
            w.tile_slot[start + i] = w.emit_slot[ee] | (e[r] & OVR_BIT);
        }
    }
#else
    warp_bitonic<R>(k, s, e, lane);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = r * 32 + lane;
        if (i < n) {
            w.tile_e[start + i] = e[r];
            w.tile_slot[start + i] = s[r];
        }
    }
#endif
}

constexpr int WARP_SORT_CAP = 256;

// Per-tile depth sort, one warp per tile (4 tiles per CTA).  Keys are
// (camera depth bits, slot); slot order is id order, so the per-tile list is
// the reference's global stable depth order restricted to the tile.  Tiles
// longer than WARP_SORT_CAP are queued for k_tile_sort_big.
__global__ void __launch_bounds__(128) k_tile_sort(Ws w) {
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (t >= w.ntiles) return;
    const int start = w.tile_start[t], n = w.tile_start[t + 1] - start;
    if (n <= 0) return;
    if (n == 1) {
        // a single entry is already in place (the scatter wrote its slot)
    } else if (n <= 32) {
        warp_sort_tile<1>(w, start, n, lane);
    } else if (n <= 64) {
        warp_sort_tile<2>(w, start, n, lane);
    } else if (n <= 128) {
        warp_sort_tile<4>(w, start, n, lane);
    } else if (n <= WARP_SORT_CAP) {
        warp_sort_tile<8>(w, start, n, lane);
    } else if (lane == 0) {
        const unsigned long long q = atomicAdd(&w.ctr[6], 1ull);
        w.big_tiles[q] = t;
    }
}

// Long tiles: one CTA per queued tile (grid-stride over the queue).  Up to
// SORT_CAP entries are bitonic-sorted in shared memory; longer lists are
// sorted as SORT_CAP chunks followed by rank-merge passes in global memory.
__global__ void __launch_bounds__(256) k_tile_sort_big(Ws w) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* sk = (uint64_t*)smem;
    int* ss = (int*)(sk + SORT_CAP);
    int* se = ss + SORT_CAP;
    const int nbig = (int)w.ctr[6];
    for (int q = blockIdx.x; q < nbig; q += gridDim.x) {
        const int t = w.big_tiles[q];
        const int start = w.tile_start[t], end = w.tile_start[t + 1];
        const int n = end - start;
        __syncthreads();
        if (n <= SORT_CAP) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int e = w.tile_e[start + i];
                const int slot = w.tile_slot[start + i];
                sk[i] = w.vkey[slot & SLOT_MASK];
                ss[i] = slot;
                se[i] = e;
            }
            __syncthreads();
            smem_bitonic(sk, ss, se, n);
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                w.tile_e[start + i] = se[i];
                w.tile_slot[start + i] = ss[i];
            }
            continue;
        }
        int* bufA = w.sort_scratch;
        int* bufB = w.sort_scratch + 4 * w.cap;
        for (int c0 = 0; c0 < n; c0 += SORT_CAP) {
            const int cn = min(SORT_CAP, n - c0);
            __syncthreads();
            for (int i = threadIdx.x; i < cn; i += blockDim.x) {
                const int e = w.tile_e[start + c0 + i];
                const int slot = w.tile_slot[start + c0 + i];
                sk[i] = w.vkey[slot & SLOT_MASK];
                ss[i] = slot;
                se[i] = e;
            }
            __syncthreads();
            smem_bitonic(sk, ss, se, cn);
            for (int i = threadIdx.x; i < cn; i += blockDim.x) {
                int* o = bufA + 4 * (int64_t)(start + c0 + i);
                *(uint64_t*)o = sk[i];
                o[2] = ss[i];
                o[3] = se[i];
            }
        }
        __syncthreads();
        int* src = bufA;
        int* dst = bufB;
        for (int run = SORT_CAP; run < n; run <<= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int r0 = (i / (2 * run)) * (2 * run);
                const bool inA = (i - r0) < run;
                const int a0 = r0, a1 = min(r0 + run, n);
                const int b0 = a1, b1 = min(r0 + 2 * run, n);
                const int* me = src + 4 * (int64_t)(start + i);
                const uint64_t mk = *(const uint64_t*)me;
                const int ms = me[2];
                int lo = inA ? b0 : a0, hi = inA ? b1 : a1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    const int* o = src + 4 * (int64_t)(start + mid);
                    if (key_less(*(const uint64_t*)o, o[2], mk, ms)) lo = mid + 1;
                    else hi = mid;
                }
                const int pos = r0 + (inA ? (i - a0) + (lo - b0) : (i - b0) + (lo - a0));
                int* d = dst + 4 * (int64_t)(start + pos);
                *(uint64_t*)d = mk;
                d[2] = ms;
                d[3] = me[3];
            }
            __syncthreads();
            int* tmp = src; src = dst; dst = tmp;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int* o = src + 4 * (int64_t)(start + i);
            w.tile_slot[start + i] = o[2];
            w.tile_e[start + i] = o[3];
        }
    }
}

size_t tile_sort_smem() { return SORT_CAP * (sizeof(uint64_t) + 2 * sizeof(int)); }

// ---- barrier-free preprocess: count, scan, emit ------------------------------
// A single-pass preprocess with a chained scan (decoupled look-back) spent
// ~60% of its stall samples in block barriers and look-back spins, and its
// spinning CTAs co-ran badly with other views' blends.  Instead: (1) every
// warp independently computes its 32 Gaussians'
// visibility and tile counts (no barrier, no record) and writes a ballot
// mask and two counts (plus its 1024-warp chunk's totals); (2) one CTA per
// chunk scans the per-warp counts from the chunk's base; (3) warps that
// hold a visible Gaussian recompute it fully (the same code, so the same
// bits) and write the records, keys and intersections at their offsets.
// Slot order is still id order.

#ifndef LSB_PRE_STASH
#define LSB_PRE_STASH 1       // the counting pass computes visible Gaussians in full and stashes them
#endif
__global__ void __launch_bounds__(PRE_THREADS) k_pre_count(PreArgs a, Ws w) {
    const int64_t i = (int64_t)blockIdx.x * PRE_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    Rec r;
    int nt = 0;
    uint64_t key = 0;
    uint32_t cm = 0;
    CullGeo geo;
    const bool vis = (i < a.p.n) && splat_one<LSB_PRE_STASH>(a, i, r, nt, key, cm, geo);
#if LSB_PRE_STASH
    if (vis) {                          // the emitting pass copies this instead of recomputing it
        w.st_rec[i] = r;
        w.st_key[i] = key;
        w.st_cm[i] = cm;
        w.st_nt[i] = nt;
        if (a.s.alpha_cut > 0.0) w.st_geo[i] = geo;
    }
#endif
    const unsigned mask = __ballot_sync(0xffffffffu, vis);
    int t = vis ? nt : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) {
        const int64_t wid = i >> 5;
        w.warp_mask[wid] = mask;
        w.warp_cnt[2 * wid] = __popc(mask);
        w.warp_cnt[2 * wid + 1] = t;
        if (mask) {                      // chunk totals for the scan (integer: order-free)
            atomicAdd(&w.chunk_cnt[2 * (wid >> 10)], __popc(mask));
            atomicAdd(&w.chunk_cnt[2 * (wid >> 10) + 1], t);
        }
    }
}

constexpr int PS_THREADS = 1024;     // preprocess warps per scan chunk (one CTA each)
// Exclusive scan of the per-warp (visible, tile) counts, one CTA per chunk
// of 1024 warps: the chunk's base is the sum of the earlier chunks' totals
// (k_pre_count adds them with integer atomics), then one block scan.  Wide
// and single-pass: every SM pulls its own slice (a one-CTA scan is bound by
// one SM's memory parallelism, ~40 us for config 5's 64K warps).
__global__ void __launch_bounds__(PS_THREADS) k_pre_scan(Ws w, int64_t nw) {
    __shared__ int s_v[PS_THREADS / 32], s_t[PS_THREADS / 32], s_pass[2];
    __shared__ long long s_base[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x, nchunk = gridDim.x;
    if (warp == 0) {                     // base = totals of the chunks before this one
        long long bv = 0, bt = 0;
        for (int k = lane; k < c; k += 32) {
            bv += w.chunk_cnt[2 * k];
            bt += w.chunk_cnt[2 * k + 1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bv += __shfl_xor_sync(0xffffffffu, bv, o);
            bt += __shfl_xor_sync(0xffffffffu, bt, o);
        }
        if (lane == 0) {
            s_base[0] = bv;
            s_base[1] = bt;
        }
    }
    const int64_t wid = (int64_t)c * PS_THREADS + tid;
    int2 cv = make_int2(0, 0);
    if (wid < nw) cv = *(const int2*)(w.warp_cnt + 2 * wid);
    int xv = cv.x, xt = cv.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(0xffffffffu, xv, o), yt = __shfl_up_sync(0xffffffffu, xt, o);
        if (lane >= o) {
            xv += yv;
            xt += yt;
        }
    }
    if (lane == 31) {
        s_v[warp] = xv;
        s_t[warp] = xt;
    }
    __syncthreads();
    if (warp == 0) {                     // exclusive scan of the warp totals
        const int tv = s_v[lane], tt = s_t[lane];
        int zv = tv, zt = tt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yv = __shfl_up_sync(0xffffffffu, zv, o), yt = __shfl_up_sync(0xffffffffu, zt, o);
            if (lane >= o) {
                zv += yv;
                zt += yt;
            }
        }
        s_v[lane] = zv - tv;
        s_t[lane] = zt - tt;
        if (lane == 31) {
            s_pass[0] = zv;
            s_pass[1] = zt;
        }
    }
    __syncthreads();
    const long long rv = s_base[0] + (xv - cv.x + s_v[warp]);
    const long long rt = s_base[1] + (xt - cv.y + s_t[warp]);
    if (wid < nw) *(int2*)(w.warp_off + 2 * wid) = make_int2((int32_t)rv, (int32_t)min(rt, 0x7fffffffll));
    if (c == nchunk - 1 && tid == 0) {
        const long long tv = s_base[0] + s_pass[0], tt = s_base[1] + s_pass[1];
        w.ctr[0] = (unsigned long long)tv;
        w.ctr[1] = (unsigned long long)tt;
        w.vis_ebase[tv] = (int32_t)min(tt, 0x7fffffffll);
        if (tt > w.cap) {
            w.ctr[2] = 1;
            *w.sticky = 1ull;          // sticky across renders until the caller clears it
        }
    }
}

__global__ void __launch_bounds__(PRE_THREADS, PRE_MIN_BLOCKS) k_pre_emit(PreArgs a, Ws w) {
    const int64_t i = (int64_t)blockIdx.x * PRE_THREADS + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t wid = i >> 5;
    if (wid * 32 >= a.p.n) return;
    const unsigned mask = w.warp_mask[wid];
    if (mask == 0) return;                                   // warp-uniform
    const bool mine = (mask >> lane) & 1u;
    Rec r;
    int nt = 0;
    uint64_t key = 0;
    uint32_t cm = 0;
    CullGeo geo;
#if LSB_PRE_STASH
    if (mine) {                                              // visible: the counting pass's result
        r = w.st_rec[i];
        key = w.st_key[i];
        cm = w.st_cm[i];
        nt = w.st_nt[i];
        if (a.s.alpha_cut > 0.0) geo = w.st_geo[i];
    }
#else
    if (mine) splat_one<true>(a, i, r, nt, key, cm, geo);   // visible: the counting pass said so
#endif
    int ex = mine ? nt : 0;                                  // exclusive scan of nt over the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ex, o);
        if (lane >= o) ex += y;
    }
    ex -= mine ? nt : 0;
    if (!mine) return;
    const int64_t slot = (int64_t)w.warp_off[2 * wid] + __popc(mask & ((1u << lane) - 1u));
    const int64_t e0 = (int64_t)w.warp_off[2 * wid + 1] + ex;
    emit_splat(a, w, r, slot, e0, nt, key, cm, geo);
}

cudaError_t launch_preprocess(const lsb_params& p, const lsb_camera& cam, const lsb_pose& T,
                              const lsb_settings& s, const Ws& w, cudaStream_t st) {
    PreArgs a{p, cam, T, s, 0, (s.bin_mode == 1 && s.alpha_cut > 0.0) ? 1 : 0, 0, nullptr};
    int deg_store = 0;
    while ((deg_store + 2) * (deg_store + 2) <= p.sh_coeffs) ++deg_store;
    a.degree = s.sh_degree < deg_store ? s.sh_degree : deg_store;
    cudaError_t err = cudaMemsetAsync(w.ctr, 0, zero_prefix_bytes(w), st);
    if (err != cudaSuccess) return err;
    {
        const int64_t nw = (p.n + 31) / 32;
        const unsigned nb = (unsigned)((p.n + PRE_THREADS - 1) / PRE_THREADS);
        if (p.n > 0) k_pre_count<<<nb, PRE_THREADS, 0, st>>>(a, w);
        k_pre_scan<<<(unsigned)((nw + PS_THREADS - 1) / PS_THREADS > 0 ? (nw + PS_THREADS - 1) / PS_THREADS : 1),
                     PS_THREADS, 0, st>>>(w, nw);
        if (p.n > 0) k_pre_emit<<<nb, PRE_THREADS, 0, st>>>(a, w);
    }
    const int st_smem = (int)sizeof(int) * (w.ntiles + w.ntiles / 32 + 1);
    if (st_smem > 48 * 1024) cudaFuncSetAttribute(k_scan_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, st_smem);
    k_scan_tiles<<<1, ST_THREADS, st_smem, st>>>(w);
    // the band search once per splat pays off on large scenes (many entries
    // per boundary row); on small ones (single-view latency, a few large
    // splats walked serially) the scatter's per-entry search is faster
    const int splat_band = (LSB_BAND_SPLAT && s.alpha_cut > 0.0 && p.n >= LSB_BAND_SPLAT_MIN_N) ? 1 : 0;
    if (splat_band)
        k_band_splats<<<8 * 148, 256, 0, st>>>(w, s.alpha_clamp, s.alpha_cut,
                                               bbox_free_lim(s.alpha_cut, s.alpha_clamp, s.footprint_sigma));
    k_scatter_emitted<<<8 * 148, 256, 0, st>>>(w, s.alpha_clamp, s.alpha_cut,
                                               bbox_free_lim(s.alpha_cut, s.alpha_clamp, s.footprint_sigma),
                                               splat_band);
    k_tile_sort<<<(w.ntiles + 3) / 4, 128, 0, st>>>(w);
    cudaFuncSetAttribute(k_tile_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile_sort_smem());
    k_tile_sort_big<<<148, 256, tile_sort_smem(), st>>>(w);
    return cudaGetLastError();
}

// raster.splat (raster.py:188-205) for a batch: the same projection,
// covariance, footprint cull and SH colour as the preprocess, per Gaussian
// i: geo[7 i ..] = visible, mu_i (2), cov_i (00, 01, 11), camera depth and
// color[3 i ..] = the clipped SH colour (visible Gaussians), all f64.
__global__ void k_splat_out(PreArgs a, double* __restrict__ out) {
    const int64_t n = a.p.n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        Rec r;
        int nt = 0;
        uint64_t key = 0;
        uint32_t cm = 0;
        CullGeo g{};
        const bool vis = splat_one<true>(a, i, r, nt, key, cm, g);
        double* o = out + 7 * i;
        o[0] = vis ? 1.0 : 0.0;
        o[1] = g.mux;
        o[2] = g.muy;
        o[3] = g.ca;
        o[4] = g.cb;
        o[5] = g.cc;
        o[6] = vis ? __longlong_as_double((long long)key) : 0.0;
    }
}

cudaError_t launch_splat(const lsb_params& p, const lsb_camera& cam, const lsb_pose& T, const lsb_settings& s,
                         double* geo, double* color, cudaStream_t st) {
    PreArgs a{p, cam, T, s, 0, 0, 1, color};
    int deg_store = 0;
    while ((deg_store + 2) * (deg_store + 2) <= p.sh_coeffs) ++deg_store;
    a.degree = s.sh_degree < deg_store ? s.sh_degree : deg_store;
    if (p.n <= 0) return cudaSuccess;
    const unsigned nb = (unsigned)((p.n + 127) / 128);
    k_splat_out<<<nb < 1184 ? nb : 1184, 128, 0, st>>>(a, geo);
    return cudaGetLastError();
}

}  // namespace lsb
