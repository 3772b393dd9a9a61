/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the splat hot path.
 *
 * A plain-C (f64, OpenMP) restatement of the reference's per-pixel CSR
 * compositing kernels in /root/reference/pkg/src/livsplat/_kernels.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline; the product path never calls it.
 *
 * Function ↔ reference map (file:line in livsplat):
 *   oracle_camera_points     raster.py:137  (mu_c = means @ R^T + t; the
 *                            OpenBLAS dgemm k=3 micro-kernel evaluates this as
 *                            fma(r2,z,fma(r1,y,r0*x)) + t, verified bit-exact
 *                            against numpy in tests/test_oracle_golden.py)
 *   oracle_csr_count/_fill   _kernels.py:21-59   build_csr
 *   oracle_forward           _kernels.py:62-119  _alpha_of + forward
 *   oracle_backward_entries  _kernels.py:122-165 backward_per_entry
 *   oracle_accumulate        _kernels.py:168-216 accumulate_splat_grads
 *   oracle_screen_grads      _kernels.py:219-269 per_entry_screen_grads
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void oracle_camera_points(const double* m, const double* R, const double* t,
                          int64_t n, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double x = m[3 * i], y = m[3 * i + 1], z = m[3 * i + 2];
        for (int j = 0; j < 3; ++j) {
            const double* r = R + 3 * j;
            out[3 * i + j] = fma(r[2], z, fma(r[1], y, r[0] * x)) + t[j];
        }
    }
}

/* Pass 1 of build_csr: per-pixel counts -> offsets (npx+1), per-splat areas ->
 * splat_offsets (m+1).  Returns the entry total. */
int64_t oracle_csr_count(const int64_t* bb, int64_t m, int64_t h, int64_t w,
                         int64_t* offsets, int64_t* splat_offsets) {
    const int64_t npx = h * w;
    memset(offsets, 0, sizeof(int64_t) * (size_t)(npx + 1));
    splat_offsets[0] = 0;
    for (int64_t s = 0; s < m; ++s) {
        const int64_t x0 = bb[4 * s], x1 = bb[4 * s + 1], y0 = bb[4 * s + 2], y1 = bb[4 * s + 3];
        splat_offsets[s + 1] = splat_offsets[s] + (x1 - x0) * (y1 - y0);
        for (int64_t y = y0; y < y1; ++y)
            for (int64_t x = x0; x < x1; ++x) offsets[y * w + x + 1] += 1;
    }
    for (int64_t p = 0; p < npx; ++p) offsets[p + 1] += offsets[p];
    return offsets[npx];
}

/* Pass 2 of build_csr: fill pixel-major entry_splat in sorted-splat order and
 * the splat-major (entry_pos, entry_pix) view of the same entries. */
void oracle_csr_fill(const int64_t* bb, int64_t m, int64_t h, int64_t w,
                     const int64_t* offsets, int64_t* entry_splat,
                     int64_t* entry_pos, int64_t* entry_pix) {
    const int64_t npx = h * w;
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(npx > 0 ? npx : 1));
    memcpy(fill, offsets, sizeof(int64_t) * (size_t)npx);
    int64_t k = 0;
    for (int64_t s = 0; s < m; ++s) {
        const int64_t x0 = bb[4 * s], x1 = bb[4 * s + 1], y0 = bb[4 * s + 2], y1 = bb[4 * s + 3];
        for (int64_t y = y0; y < y1; ++y) {
            for (int64_t x = x0; x < x1; ++x) {
                const int64_t p = y * w + x;
                const int64_t pos = fill[p]++;
                entry_splat[pos] = s;
                entry_pos[k] = pos;
                entry_pix[k] = p;
                ++k;
            }
        }
    }
    free(fill);
}

/* Front-to-back compositing over each pixel's depth-ordered CSR list. */
void oracle_forward(const int64_t* offsets, const int64_t* entry_splat,
                    const double* mu, const double* con, const double* opac,
                    const double* col, const double* bg, int64_t h, int64_t w,
                    double clamp, double t_min, double cut,
                    double* image, double* t_final, int64_t* n_proc,
                    double* g_scr, double* a_scr, double* t_scr) {
    const int64_t npx = h * w;
    const int64_t total = offsets[npx];
    memset(g_scr, 0, sizeof(double) * (size_t)total);
    memset(a_scr, 0, sizeof(double) * (size_t)total);
    memset(t_scr, 0, sizeof(double) * (size_t)total);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t p = 0; p < npx; ++p) {
        const double ux = (double)(p % w), uy = (double)(p / w);
        double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
        int64_t count = 0;
        for (int64_t i = offsets[p]; i < offsets[p + 1]; ++i) {
            if (T < t_min) break;
            const int64_t s = entry_splat[i];
            const double dx = ux - mu[2 * s], dy = uy - mu[2 * s + 1];
            const double q = con[3 * s] * dx * dx + 2.0 * con[3 * s + 1] * dx * dy +
                             con[3 * s + 2] * dy * dy;
            const double g = exp(-0.5 * q);
            double a = opac[s] * g;
            if (a > clamp) a = clamp;
            ++count;
            if (a < cut) continue;
            g_scr[i] = g;
            a_scr[i] = a;
            t_scr[i] = T;
            const double wgt = T * a;
            c0 += wgt * col[3 * s];
            c1 += wgt * col[3 * s + 1];
            c2 += wgt * col[3 * s + 2];
            T = T * (1.0 - a);
        }
        image[3 * p] = c0 + T * bg[0];
        image[3 * p + 1] = c1 + T * bg[1];
        image[3 * p + 2] = c2 + T * bg[2];
        t_final[p] = T;
        n_proc[p] = count;
    }
}

/* Back-to-front per-entry d(loss)/d(alpha) and blend weights, selected pixels. */
void oracle_backward_entries(const int64_t* offsets, const int64_t* entry_splat,
                             const int64_t* n_proc, const double* t_final,
                             const double* gimg, const double* col, const double* bg,
                             const double* a_scr, const double* t_scr, int64_t h,
                             int64_t w, const uint8_t* sel, double* d_alpha,
                             double* w_out) {
    const int64_t npx = h * w;
    const int64_t total = offsets[npx];
    memset(d_alpha, 0, sizeof(double) * (size_t)total);
    memset(w_out, 0, sizeof(double) * (size_t)total);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t p = 0; p < npx; ++p) {
        if (!sel[p] || n_proc[p] == 0) continue;
        const double g0 = gimg[3 * p], g1 = gimg[3 * p + 1], g2 = gimg[3 * p + 2];
        double s0 = bg[0] * t_final[p], s1 = bg[1] * t_final[p], s2 = bg[2] * t_final[p];
        for (int64_t k = n_proc[p] - 1; k >= 0; --k) {
            const int64_t pos = offsets[p] + k;
            const double a = a_scr[pos];
            if (a == 0.0) continue;
            const int64_t s = entry_splat[pos];
            const double Ti = t_scr[pos];
            const double wgt = a * Ti;
            const double inv = 1.0 / (1.0 - a);
            double da = g0 * (col[3 * s] * Ti - s0 * inv);
            da += g1 * (col[3 * s + 1] * Ti - s1 * inv);
            da += g2 * (col[3 * s + 2] * Ti - s2 * inv);
            d_alpha[pos] = da;
            w_out[pos] = wgt;
            s0 += wgt * col[3 * s];
            s1 += wgt * col[3 * s + 1];
            s2 += wgt * col[3 * s + 2];
        }
    }
}

/* Race-free per-splat accumulation of screen-space gradients. */
void oracle_accumulate(const int64_t* splat_offsets, int64_t m, const int64_t* entry_pos,
                       const int64_t* entry_pix, const double* d_alpha, const double* w_out,
                       const double* g_scr, const double* a_scr, const double* gimg,
                       const double* mu, const double* con, const double* opac, int64_t w,
                       double clamp, double* d_color, double* d_opac, double* d_mu,
                       double* d_cov) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t s = 0; s < m; ++s) {
        double dc0 = 0, dc1 = 0, dc2 = 0, dop = 0, dm0 = 0, dm1 = 0, dv0 = 0, dv1 = 0, dv2 = 0;
        const double mx = mu[2 * s], my = mu[2 * s + 1];
        const double ca = con[3 * s], cb = con[3 * s + 1], cc = con[3 * s + 2], op = opac[s];
        for (int64_t k = splat_offsets[s]; k < splat_offsets[s + 1]; ++k) {
            const int64_t pos = entry_pos[k];
            const double da = d_alpha[pos], wg = w_out[pos];
            if (da == 0.0 && wg == 0.0) continue;
            const int64_t p = entry_pix[k];
            dc0 += wg * gimg[3 * p];
            dc1 += wg * gimg[3 * p + 1];
            dc2 += wg * gimg[3 * p + 2];
            if (a_scr[pos] < clamp) {
                const double g = g_scr[pos];
                const double dx = (double)(p % w) - mx, dy = (double)(p / w) - my;
                dop += g * da;
                const double gg = op * da * g;
                const double v0 = ca * dx + cb * dy, v1 = cb * dx + cc * dy;
                dm0 += gg * v0;
                dm1 += gg * v1;
                dv0 += 0.5 * gg * v0 * v0;
                dv1 += 0.5 * gg * v0 * v1;
                dv2 += 0.5 * gg * v1 * v1;
            }
        }
        d_color[3 * s] = dc0; d_color[3 * s + 1] = dc1; d_color[3 * s + 2] = dc2;
        d_opac[s] = dop;
        d_mu[2 * s] = dm0; d_mu[2 * s + 1] = dm1;
        d_cov[3 * s] = dv0; d_cov[3 * s + 1] = dv1; d_cov[3 * s + 2] = dv2;
    }
}

/* Per-entry screen-space pieces for selected pixels (pose rows).  keep[k]=1 for
 * entries that contribute; mu (2), cov (3), w and the splat/pixel ids. */
void oracle_screen_grads(int64_t total, const int64_t* entry_pos, const int64_t* entry_pix,
                         const int64_t* entry_splat, const double* d_alpha,
                         const double* w_out, const double* g_scr, const double* a_scr,
                         const double* mu, const double* con, const double* opac,
                         int64_t w, double clamp, const uint8_t* sel, uint8_t* keep,
                         int64_t* o_splat, int64_t* o_pix, double* o_mu, double* o_cov,
                         double* o_w) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < total; ++k) {
        keep[k] = 0;
        o_splat[k] = 0; o_pix[k] = 0; o_w[k] = 0;
        o_mu[2 * k] = o_mu[2 * k + 1] = 0;
        o_cov[3 * k] = o_cov[3 * k + 1] = o_cov[3 * k + 2] = 0;
        const int64_t p = entry_pix[k];
        if (!sel[p]) continue;
        const int64_t pos = entry_pos[k];
        const double da = d_alpha[pos], wg = w_out[pos];
        if (da == 0.0 && wg == 0.0) continue;
        const int64_t s = entry_splat[pos];
        keep[k] = 1;
        o_splat[k] = s;
        o_pix[k] = p;
        o_w[k] = wg;
        if (a_scr[pos] < clamp) {
            const double dx = (double)(p % w) - mu[2 * s], dy = (double)(p / w) - mu[2 * s + 1];
            const double ca = con[3 * s], cb = con[3 * s + 1], cc = con[3 * s + 2];
            const double gg = opac[s] * da * g_scr[pos];
            const double v0 = ca * dx + cb * dy, v1 = cb * dx + cc * dy;
            o_mu[2 * k] = gg * v0;
            o_mu[2 * k + 1] = gg * v1;
            o_cov[3 * k] = 0.5 * gg * v0 * v0;
            o_cov[3 * k + 1] = 0.5 * gg * v0 * v1;
            o_cov[3 * k + 2] = 0.5 * gg * v1 * v1;
        }
    }
}
