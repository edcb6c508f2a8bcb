// basis.cuh -- host-side construction of the DGSEM N=3 tables.
//
// Independent of the test oracle: LGL weights from w_i = 2 / (N (N+1) P_N(xi_i)^2); derivative matrix and
// interpolation from the barycentric formulas; the exact L2 mortar projection from the orthonormal
// Legendre Vandermonde V (mass matrix M = (V V^T)^{-1}):  R_half = 1/2 M^{-1} P_half^T M.
#pragma once
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace perk {

static double legendre(int n, double x)
{
    double p0 = 1.0, p1 = x;
    if (n == 0) return p0;
    for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
    }
    return p1;
}

static void barycentric_weights(const double *xi, double *lam)
{
    for (int j = 0; j < NP; ++j) {
        double p = 1.0;
        for (int k = 0; k < NP; ++k)
            if (k != j) p *= (xi[j] - xi[k]);
        lam[j] = 1.0 / p;
    }
}

// all Lagrange basis values l_j(x), barycentric form 2 (exact at the nodes)
static void lagrange_all(const double *xi, const double *lam, double x, double *out)
{
    for (int j = 0; j < NP; ++j)
        if (x == xi[j]) {
            for (int k = 0; k < NP; ++k) out[k] = k == j ? 1.0 : 0.0;
            return;
        }
    double den = 0.0;
    for (int k = 0; k < NP; ++k) den += lam[k] / (x - xi[k]);
    for (int j = 0; j < NP; ++j) out[j] = lam[j] / (x - xi[j]) / den;
}

static bool invert4(const double A[NP][NP], double Ainv[NP][NP])  // Gauss-Jordan
{
    double M[NP][2 * NP];
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < 2 * NP; ++j) M[i][j] = j < NP ? A[i][j] : (j - NP == i ? 1.0 : 0.0);
    for (int c = 0; c < NP; ++c) {
        int p = c;
        for (int r = c + 1; r < NP; ++r)
            if (std::fabs(M[r][c]) > std::fabs(M[p][c])) p = r;
        if (M[p][c] == 0.0) return false;
        for (int j = 0; j < 2 * NP; ++j) std::swap(M[c][j], M[p][j]);
        double d = M[c][c];
        for (int j = 0; j < 2 * NP; ++j) M[c][j] /= d;
        for (int r = 0; r < NP; ++r)
            if (r != c) {
                double f = M[r][c];
                for (int j = 0; j < 2 * NP; ++j) M[r][j] -= f * M[c][j];
            }
    }
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) Ainv[i][j] = M[i][j + NP];
    return true;
}

static void build_basis(BasisTables &B)
{
    const int N = NP - 1;
    const double s = 1.0 / std::sqrt(5.0);
    const double xi[NP] = {-1.0, -s, s, 1.0};  // roots of (1 - x^2) P_3'(x)
    for (int i = 0; i < NP; ++i) {
        B.xi[i] = xi[i];
        double pn = legendre(N, xi[i]);
        B.w[i] = 2.0 / (N * (N + 1.0) * pn * pn);
        B.invw[i] = 1.0 / B.w[i];
    }
    double lam[NP];
    barycentric_weights(xi, lam);
    double D[NP][NP];
    for (int i = 0; i < NP; ++i) {
        double diag = 0.0;
        for (int j = 0; j < NP; ++j)
            if (j != i) {
                D[i][j] = (lam[j] / lam[i]) / (xi[i] - xi[j]);
                diag -= D[i][j];
            }
        D[i][i] = diag;
    }
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) {
            B.Dhat[i][j] = B.w[j] * D[j][i] / B.w[i];
            B.Dsplit[i][j] = 2.0 * D[i][j];
        }
    B.Dsplit[0][0] += 1.0 / B.w[0];
    B.Dsplit[N][N] -= 1.0 / B.w[N];
    for (int i = 0; i < NP; ++i) {
        lagrange_all(xi, lam, 0.5 * (xi[i] - 1.0), B.Plo[i]);
        lagrange_all(xi, lam, 0.5 * (xi[i] + 1.0), B.Pup[i]);
    }
    // orthonormal Legendre Vandermonde and the exact mass matrix
    double V[NP][NP], VVt[NP][NP], M[NP][NP];
    for (int i = 0; i < NP; ++i)
        for (int k = 0; k < NP; ++k) V[i][k] = std::sqrt((2.0 * k + 1.0) / 2.0) * legendre(k, xi[i]);
    for (int i = 0; i < NP; ++i)
        for (int j = 0; j < NP; ++j) {
            double a = 0.0;
            for (int k = 0; k < NP; ++k) a += V[i][k] * V[j][k];
            VVt[i][j] = a;   // = M^{-1}
        }
    invert4(VVt, M);
    invert4(V, B.Vinv);
    std::memcpy(B.D, D, sizeof(D));
    for (int half = 0; half < 2; ++half) {
        const double (*P)[NP] = half == 0 ? B.Plo : B.Pup;
        double (*R)[NP] = half == 0 ? B.Rlo : B.Rup;
        double PtM[NP][NP];
        for (int i = 0; i < NP; ++i)
            for (int j = 0; j < NP; ++j) {
                double a = 0.0;
                for (int k = 0; k < NP; ++k) a += P[k][i] * M[k][j];
                PtM[i][j] = a;
            }
        for (int i = 0; i < NP; ++i)
            for (int j = 0; j < NP; ++j) {
                double a = 0.0;
                for (int k = 0; k < NP; ++k) a += VVt[i][k] * PtM[k][j];
                R[i][j] = 0.5 * a;
            }
    }
}

}  // namespace perk
