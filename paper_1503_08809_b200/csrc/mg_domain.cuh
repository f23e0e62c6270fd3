// mg_domain.cuh — the tetrahedral l-triple domain and its weights.
//
// Reference: geometry.py:145-200 (TriangularDomain: l1 outer, l2 >= l1, l3 from l2 (l1 even)
// or l2+1 (l1 odd) in steps of 2 up to min(l1+l2, l_max)), geometry.py:89-142 (Gosper h^2,
// geometric prefactor), geometry.py:114-123 (multiplicity), engine3d.py:41-53,133-134 (zm).
//
// The domain is never materialised: flat index <-> triple goes through (l1,l2)-row prefix
// sums (36 MB at l_max = 3000 instead of the reference's 27 GB of int64 arrays).
//
// Bit-exactness: every FP64 operation of the Gosper weight is an explicit round-to-nearest
// intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn), so no FMA contraction can happen and
// the evaluation order is NumPy's left-to-right order.
#pragma once

#include <cstdint>
#include <vector>

namespace mg {

// Triples in the reference's (l1,l2) row: l3 = start, start+2, ..., <= min(l1+l2, l_max).
__host__ __device__ inline int row_len(int l1, int l2, int l_max) {
    int start = ((l1 & 1) == 0) ? l2 : l2 + 1;  // (l1 + 2 l2) even  <=>  l1 even
    int stop = (l1 + l2 < l_max) ? l1 + l2 : l_max;
    return start > stop ? 0 : (stop - start) / 2 + 1;
}
__host__ __device__ inline int row_start(int l1, int l2) { return ((l1 & 1) == 0) ? l2 : l2 + 1; }

// Host-side prefix tables of the reference enumeration.
struct DomainIndex {
    int l_min = 2, l_max = 2;
    std::vector<int64_t> l1_base;   // [L+1] first flat index of each l1
    std::vector<int64_t> row_base;  // [rows+1] first flat index of each (l1,l2) pair, l2>=l1
    std::vector<int64_t> pair_off;  // [L+1] position of (l1, l2=l1) in row_base
    int64_t count = 0;
    int64_t nonempty_rows = 0;

    void build(int lmin, int lmax) {
        l_min = lmin;
        l_max = lmax;
        int L = lmax - lmin + 1;
        l1_base.assign(L + 1, 0);
        pair_off.assign(L + 1, 0);
        row_base.clear();
        row_base.reserve((size_t)L * (L + 1) / 2 + 1);
        int64_t t = 0;
        nonempty_rows = 0;
        for (int l1 = lmin; l1 <= lmax; ++l1) {
            l1_base[l1 - lmin] = t;
            pair_off[l1 - lmin] = (int64_t)row_base.size();
            for (int l2 = l1; l2 <= lmax; ++l2) {
                row_base.push_back(t);
                int n = row_len(l1, l2, lmax);
                nonempty_rows += n > 0;
                t += n;
            }
        }
        l1_base[L] = t;
        pair_off[L] = (int64_t)row_base.size();
        row_base.push_back(t);
        count = t;
    }

    // Triple at flat index idx (0 <= idx < count); idx == count gives the sentinel
    // (l_max+1, 0, 0) which compares greater than every triple.
    void triple(int64_t idx, int& l1, int& l2, int& l3) const {
        if (idx >= count) {
            l1 = l_max + 1; l2 = 0; l3 = 0;
            return;
        }
        int L = l_max - l_min + 1;
        int lo = 0, hi = L;  // find last l1 with base <= idx
        while (hi - lo > 1) {
            int mid = (lo + hi) / 2;
            if (l1_base[mid] <= idx) lo = mid; else hi = mid;
        }
        l1 = l_min + lo;
        int64_t a = pair_off[lo], b = pair_off[lo + 1];  // rows of this l1: [a, b)
        while (b - a > 1) {
            int64_t mid = (a + b) / 2;
            if (row_base[mid] <= idx) a = mid; else b = mid;
        }
        // skip empty rows that share the same base (take the row that contains idx)
        while (a + 1 < pair_off[lo + 1] && row_base[a + 1] <= idx) ++a;
        l2 = l1 + (int)(a - pair_off[lo]);
        l3 = row_start(l1, l2) + 2 * (int)(idx - row_base[a]);
    }
};

__host__ __device__ inline int multiplicity(int l1, int l2, int l3) {
    return (l1 == l3) ? 1 : ((l1 == l2 || l2 == l3) ? 3 : 6);
}

#ifdef __CUDACC__
// h2_gosper(l1,l2,l3) / (36 v1 v2 v3 sqrt(C1 C2 C3)) * mult, NumPy-order, no contraction.
__device__ __forceinline__ double zm_gosper(int l1, int l2, int l3, const double* __restrict__ C,
                                            const double* __restrict__ v, int l_min) {
    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    const double two_pi2 = 2.0 * 9.869604401089358;
    double a = (double)l1, b = (double)l2, c = (double)l3;
    double L = __dadd_rn(__dadd_rn(a, b), c);
    double La = __dsub_rn(L, __dmul_rn(2.0, a));
    double Lb = __dsub_rn(L, __dmul_rn(2.0, b));
    double Lc = __dsub_rn(L, __dmul_rn(2.0, c));
    double na = __dadd_rn(__dmul_rn(2.0, a), 1.0);
    double nb = __dadd_rn(__dmul_rn(2.0, b), 1.0);
    double nc = __dadd_rn(__dmul_rn(2.0, c), 1.0);
    double num = __dmul_rn(__dmul_rn(__dmul_rn(na, nb), nc), __dadd_rn(L, third));
    double den = __dmul_rn(__dmul_rn(__dmul_rn(__dadd_rn(L, 1.0), __dadd_rn(La, third)),
                                     __dadd_rn(Lb, third)),
                           __dadd_rn(Lc, third));
    double mainv = __ddiv_rn(num, den);
    double rad = __ddiv_rn(__dmul_rn(__dmul_rn(__dadd_rn(La, sixth), __dadd_rn(Lb, sixth)),
                                     __dadd_rn(Lc, sixth)),
                           __dadd_rn(L, sixth));
    double h2 = __ddiv_rn(__dmul_rn(mainv, __dsqrt_rn(rad)), two_pi2);
    int i1 = l1 - l_min, i2 = l2 - l_min, i3 = l3 - l_min;
    double denom = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(36.0, v[i1]), v[i2]), v[i3]),
                             __dsqrt_rn(__dmul_rn(__dmul_rn(C[i1], C[i2]), C[i3])));
    return __dmul_rn(__ddiv_rn(h2, denom), (double)multiplicity(l1, l2, l3));
}

// h2_exact via a log-factorial table lf[] (geometry.py:73-85), then the same prefactor.
// Like the reference (theta_indicator gate, geometry.py:44-54,67-71) the weight is exactly 0
// where the triangle or even-parity condition fails — the sparse config-3 domain and explicit
// triple lists may contain such triples, and the log-factorial indices are invalid there.
__device__ __forceinline__ double zm_exact(int l1, int l2, int l3, const double* __restrict__ C,
                                           const double* __restrict__ v, int l_min,
                                           const double* __restrict__ lf) {
    const double four_pi = 4.0 * 3.141592653589793;
    int L = l1 + l2 + l3, g = L / 2;
    if ((L & 1) || l3 > l1 + l2 || l2 > l1 + l3 || l1 > l2 + l3) return 0.0;
    double s = __dsub_rn(__dadd_rn(__dadd_rn(lf[L - 2 * l1], lf[L - 2 * l2]), lf[L - 2 * l3]),
                         lf[L + 1]);
    double t = __dsub_rn(__dsub_rn(__dsub_rn(lf[g], lf[g - l1]), lf[g - l2]), lf[g - l3]);
    double log3j2 = __dadd_rn(s, __dmul_rn(2.0, t));
    long long pi = (long long)(2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1);
    double pref = __ddiv_rn((double)pi, four_pi);
    double h2 = __dmul_rn(pref, exp(log3j2));
    int i1 = l1 - l_min, i2 = l2 - l_min, i3 = l3 - l_min;
    double denom = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(36.0, v[i1]), v[i2]), v[i3]),
                             __dsqrt_rn(__dmul_rn(__dmul_rn(C[i1], C[i2]), C[i3])));
    return __dmul_rn(__ddiv_rn(h2, denom), (double)multiplicity(l1, l2, l3));
}

// Same quantity as zm_gosper, factored for the Γ pipeline (not bit-identical to NumPy, equal
// to it within a few ulp): zm = mult/(72 π²) · f(l1) f(l2) f(l3) · g(L, L1, L2, L3),
// f(l) = (2l+1)/(v_l sqrt C_l) (table fl[] indexed l - l_min),
// g = (L+1/3) sqrt((L1+1/6)(L2+1/6)(L3+1/6)(L+1/6)) / ((L+1)(L1+1/3)(L2+1/3)(L3+1/3)(L+1/6)).
__device__ __forceinline__ double zm_gosper_fast(int l1, int l2, int l3,
                                                 const double* __restrict__ fl, int l_min) {
    const double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    const double inv72pi2 = 1.0 / (72.0 * 9.869604401089358);
    const double L = (double)(l1 + l2 + l3);
    const double La = (double)(l2 + l3 - l1), Lb = (double)(l1 + l3 - l2),
                 Lc = (double)(l1 + l2 - l3);
    const double s = (La + sixth) * (Lb + sixth) * (Lc + sixth) * (L + sixth);
    const double den = (L + 1.0) * (La + third) * (Lb + third) * (Lc + third) * (L + sixth);
    const double g = (L + third) * sqrt(s) / den;
    return (double)multiplicity(l1, l2, l3) * inv72pi2 * fl[l1 - l_min] * fl[l2 - l_min] *
           fl[l3 - l_min] * g;
}

__device__ __forceinline__ double zm_weight(int mode, int l1, int l2, int l3,
                                            const double* __restrict__ C,
                                            const double* __restrict__ v, int l_min,
                                            const double* __restrict__ lf) {
    return mode == 0 ? zm_gosper(l1, l2, l3, C, v, l_min)
                     : zm_exact(l1, l2, l3, C, v, l_min, lf);
}
#endif

}  // namespace mg
