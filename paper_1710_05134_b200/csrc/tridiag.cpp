// tridiag.cpp — host symmetric tridiagonal eigensolver for the Lanczos stages
// (Eq. (2.2) T_j y = theta y of Alg. 2; Eq. (2.5) of Alg. 3,
// PAPER.md:153-157; "host, tiny": j is at most a few hundred).
//
// Implicit symmetric QR with the Wilkinson shift (Golub & Van Loan, "Matrix
// Computations", Alg. 8.3.2 / 8.3.3): on the unreduced diagonal block [p, q]
// the first Givens rotation is chosen from (t_pp - mu, t_p+1,p), mu the
// eigenvalue of the trailing 2x2 closer to t_qq, and the bulge it creates is
// chased down the band; off-diagonals with |e_i| <= eps (|d_i| + |d_i+1|) are
// set to zero (deflation).  The rotations are accumulated in Z, so
// T = Z diag(d) Z^T on return, eigenvalues ascending.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

namespace kep {

bool tridiag_eigen(std::vector<double>& d, std::vector<double> e, std::vector<double>& Z) {
    const int n = (int)d.size();
    Z.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) Z[i + (size_t)i * n] = 1.0;
    if (n <= 1) return true;
    e.resize(n - 1, 0.0);
    int q = n - 1;                 // the block [q+1, n) is diagonal
    long iters = 0;
    const long max_iters = 64L * n;
    while (q > 0) {
        for (int i = 0; i < q; ++i)                                   // deflation
            if (std::fabs(e[i]) <= DBL_EPSILON * (std::fabs(d[i]) + std::fabs(d[i + 1]))) e[i] = 0.0;
        while (q > 0 && e[q - 1] == 0.0) --q;
        if (q == 0) break;
        int p = q - 1;                                                // unreduced block [p, q]
        while (p > 0 && e[p - 1] != 0.0) --p;
        if (++iters > max_iters) return false;
        // Wilkinson shift from the trailing 2x2 of the block
        const double dd = 0.5 * (d[q - 1] - d[q]), bq = e[q - 1];
        const double den = dd + std::copysign(std::hypot(dd, bq), dd == 0.0 ? 1.0 : dd);
        const double mu = d[q] - bq * bq / den;
        double x = d[p] - mu, z = e[p];
        for (int k = p; k < q; ++k) {
            // rotation R = [c s; -s c] on (k, k+1) with R [x; z] = [r; 0]
            const double r = std::hypot(x, z);
            double c = 1.0, s = 0.0;
            if (r != 0.0) { c = x / r; s = z / r; }
            if (k > p) e[k - 1] = r;                                  // the bulge is gone from row k+1
            const double ak = d[k], ak1 = d[k + 1], bk = e[k];
            d[k] = c * c * ak + 2.0 * c * s * bk + s * s * ak1;
            d[k + 1] = s * s * ak - 2.0 * c * s * bk + c * c * ak1;
            e[k] = c * s * (ak1 - ak) + (c * c - s * s) * bk;
            if (k + 1 < q) {                                          // new bulge at (k+2, k)
                x = e[k];
                z = s * e[k + 1];
                e[k + 1] *= c;
            }
            double* zk = &Z[(size_t)k * n];
            double* zk1 = &Z[(size_t)(k + 1) * n];
            for (int i = 0; i < n; ++i) {                             // Z <- Z R^T
                const double a = zk[i], b = zk1[i];
                zk[i] = c * a + s * b;
                zk1[i] = -s * a + c * b;
            }
        }
    }
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
    std::vector<double> d2(n), Z2((size_t)n * n);
    for (int k = 0; k < n; ++k) {
        d2[k] = d[idx[k]];
        std::memcpy(&Z2[(size_t)k * n], &Z[(size_t)idx[k] * n], sizeof(double) * n);
    }
    d.swap(d2);
    Z.swap(Z2);
    return true;
}

}  // namespace kep

// Testing hook (include/kep.h): the same solver through the C ABI.
#include "../../include/kep.h"
extern "C" kep_status kep_tridiag_eigen(int32_t n, const double* d, const double* e, double* w, double* Z) {
    if (n < 0 || (n > 0 && (!d || !w || !Z)) || (n > 1 && !e)) return KEP_EINVAL;
    std::vector<double> dd(d, d + n), ee(n > 1 ? e : d, n > 1 ? e + n - 1 : d), zz;
    if (!kep::tridiag_eigen(dd, ee, zz)) return KEP_ENOCONV;
    std::memcpy(w, dd.data(), sizeof(double) * n);
    std::memcpy(Z, zz.data(), sizeof(double) * (size_t)n * n);
    return KEP_OK;
}
