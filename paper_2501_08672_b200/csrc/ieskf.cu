// Host-side 15x15 gain algebra of one IESKF iteration (estimator.py:292-331,
// the `ieskf_update` loop body) for the visual update, whose H has only its
// six pose columns non-zero: with A = H^T R^-1 H (6x6 block) and b = H^T R^-1 z
// from lsb_hb_reduce / lsb_visual_pass,
//   P  = Hj^-1 cov Hj^-T        (Hj^-1 = I with J_l(-d_rho) in the rotation block)
//   S  = A + P^-1,  K H = S^-1 A,  K z = S^-1 b
//   xi = -K z - (I - K H) Hj^-1 delta
// Plain C++ on the host (15x15: a few thousand flops); Gauss-Jordan with
// partial pivoting for the two inverses (the reference calls LAPACK through
// numpy.linalg.inv: the results agree to round-off).
#include <math.h>
#include <string.h>

namespace lsb {

constexpr int DIM = 15;

// In-place inverse of the n x n row-major matrix m; false if singular.
static bool invert(double* m, int n) {
    double inv[DIM * DIM];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) inv[i * n + j] = i == j ? 1.0 : 0.0;
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabs(m[r * n + c]) > fabs(m[piv * n + c])) piv = r;
        if (m[piv * n + c] == 0.0 || !isfinite(m[piv * n + c])) return false;
        if (piv != c)
            for (int j = 0; j < n; ++j) {
                double t = m[c * n + j];
                m[c * n + j] = m[piv * n + j];
                m[piv * n + j] = t;
                t = inv[c * n + j];
                inv[c * n + j] = inv[piv * n + j];
                inv[piv * n + j] = t;
            }
        const double d = 1.0 / m[c * n + c];
        for (int j = 0; j < n; ++j) {
            m[c * n + j] *= d;
            inv[c * n + j] *= d;
        }
        for (int r = 0; r < n; ++r) {
            if (r == c) continue;
            const double f = m[r * n + c];
            if (f == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                m[r * n + j] -= f * m[c * n + j];
                inv[r * n + j] -= f * inv[c * n + j];
            }
        }
    }
    memcpy(m, inv, sizeof(double) * n * n);
    return true;
}

static void matmul(const double* a, const double* b, double* c) {
    for (int i = 0; i < DIM; ++i)
        for (int j = 0; j < DIM; ++j) {
            double s = 0.0;
            for (int k = 0; k < DIM; ++k) s += a[i * DIM + k] * b[k * DIM + j];
            c[i * DIM + j] = s;
        }
}

// 0 ok, 1 singular (P or S), 2 non-finite gain
int ieskf_gain(const double* cov, const double* jinv3, const double* A6, const double* b6, const double* delta,
               double* xi, double* KH, double* P) {
    double H[DIM * DIM], T[DIM * DIM], Ht[DIM * DIM];
    for (int i = 0; i < DIM; ++i)
        for (int j = 0; j < DIM; ++j) H[i * DIM + j] = i == j ? 1.0 : 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) H[i * DIM + j] = jinv3[3 * i + j];
    for (int i = 0; i < DIM; ++i)
        for (int j = 0; j < DIM; ++j) Ht[i * DIM + j] = H[j * DIM + i];
    matmul(H, cov, T);
    matmul(T, Ht, P);
    double S[DIM * DIM];
    memcpy(S, P, sizeof(S));
    if (!invert(S, DIM)) return 1;
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) S[i * DIM + j] += A6[6 * i + j];
    if (!invert(S, DIM)) return 1;                         // S^-1
    for (int i = 0; i < DIM; ++i)
        for (int j = 0; j < DIM; ++j) {
            double s = 0.0;
            if (j < 6)
                for (int k = 0; k < 6; ++k) s += S[i * DIM + k] * A6[6 * k + j];
            KH[i * DIM + j] = s;
            if (!isfinite(s)) return 2;
        }
    double hd[DIM];
    for (int i = 0; i < DIM; ++i) {
        double s = 0.0;
        for (int k = 0; k < DIM; ++k) s += H[i * DIM + k] * delta[k];
        hd[i] = s;
    }
    for (int i = 0; i < DIM; ++i) {
        double kz = 0.0;
        for (int k = 0; k < 6; ++k) kz += S[i * DIM + k] * b6[k];
        double r = 0.0;
        for (int k = 0; k < DIM; ++k) r += ((i == k ? 1.0 : 0.0) - KH[i * DIM + k]) * hd[k];
        xi[i] = -kz - r;
    }
    return 0;
}

}  // namespace lsb
