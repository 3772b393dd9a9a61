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
#define _USE_MATH_DEFINES
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

// ---- SO(3) helpers (geometry.py: so3_exp / so3_log / so3_left_jacobian) ----
static void hat3(const double* v, double* S) {
    S[0] = 0.0;   S[1] = -v[2]; S[2] = v[1];
    S[3] = v[2];  S[4] = 0.0;   S[5] = -v[0];
    S[6] = -v[1]; S[7] = v[0];  S[8] = 0.0;
}
static void mul3(const double* a, const double* b, double* c) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}
static void so3_exp3(const double* phi, double* E) {
    const double th = sqrt(phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2]);
    double S[9], SS[9];
    hat3(phi, S);
    mul3(S, S, SS);
    const double a = th < 1e-8 ? 1.0 : sin(th) / th, b = th < 1e-8 ? 0.5 : (1.0 - cos(th)) / (th * th);
    for (int k = 0; k < 9; ++k) E[k] = (k % 4 == 0 ? 1.0 : 0.0) + a * S[k] + b * SS[k];
}
static void so3_log3(const double* R, double* w) {
    double c = 0.5 * (R[0] + R[4] + R[8] - 1.0);
    c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
    const double th = acos(c);
    const double v[3] = {R[7] - R[5], R[2] - R[6], R[3] - R[1]};
    if (th < 1e-8) {
        for (int k = 0; k < 3; ++k) w[k] = 0.5 * v[k];
        return;
    }
    if (M_PI - th > 1e-6) {
        const double f = th / (2.0 * sin(th));
        for (int k = 0; k < 3; ++k) w[k] = f * v[k];
        return;
    }
    double B[9];
    for (int k = 0; k < 9; ++k) B[k] = 0.5 * (R[k] + (k % 4 == 0 ? 1.0 : 0.0));
    int kk = 0;
    for (int k = 1; k < 3; ++k)
        if (B[4 * k] > B[4 * kk]) kk = k;
    const double d = sqrt(B[4 * kk] > 1e-12 ? B[4 * kk] : 1e-12);
    double ax[3] = {B[kk] / d, B[3 + kk] / d, B[6 + kk] / d};
    const double n = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    for (int k = 0; k < 3; ++k) ax[k] /= n;
    if (v[0] * ax[0] + v[1] * ax[1] + v[2] * ax[2] < 0.0)
        for (int k = 0; k < 3; ++k) ax[k] = -ax[k];
    for (int k = 0; k < 3; ++k) w[k] = th * ax[k];
}
static void so3_jl3(const double* phi, double* J) {
    const double th = sqrt(phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2]);
    double S[9], SS[9];
    hat3(phi, S);
    mul3(S, S, SS);
    double a, b;
    if (th < 1e-6) {
        a = 0.5;
        b = 1.0 / 6.0;
    } else {
        a = (1.0 - cos(th)) / (th * th);
        b = (th - sin(th)) / (th * th * th);
    }
    for (int k = 0; k < 9; ++k) J[k] = (k % 4 == 0 ? 1.0 : 0.0) + a * S[k] + b * SS[k];
}

// One iteration of the visual IESKF update on the state vectors
// x = [R (9, row-major) | t | v | bg | ba] (21 doubles): delta = x_hat [-] x_bar
// (NavState.boxminus), the gain algebra above, x_hat <- x_hat [+] xi
// (NavState.boxplus with the bias clip).  Returns ieskf_gain's code.
int ieskf_iterate(const double* cov, const double* xbar, double* xhat, const double* A6, const double* b6,
                  double bias_limit, double* xi, double* KH, double* P) {
    double delta[DIM], Rt[9], RtR[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Rt[3 * i + j] = xbar[3 * j + i];
    mul3(Rt, xhat, RtR);
    so3_log3(RtR, delta);
    for (int k = 3; k < DIM; ++k) delta[k] = xhat[6 + k] - xbar[6 + k];
    const double mrho[3] = {-delta[0], -delta[1], -delta[2]};
    double J[9];
    so3_jl3(mrho, J);
    const int rc = ieskf_gain(cov, J, A6, b6, delta, xi, KH, P);
    if (rc) return rc;
    double E[9], Rn[9];
    so3_exp3(xi, E);
    mul3(xhat, E, Rn);
    for (int k = 0; k < 9; ++k) xhat[k] = Rn[k];
    for (int k = 3; k < 9; ++k) xhat[6 + k] += xi[k];
    for (int k = 9; k < DIM; ++k) {
        const double b = xhat[6 + k] + xi[k];
        xhat[6 + k] = b < -bias_limit ? -bias_limit : (b > bias_limit ? bias_limit : b);
    }
    return 0;
}

}  // namespace lsb
