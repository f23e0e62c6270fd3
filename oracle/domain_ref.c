/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain-C restatement of the reference's l-triple enumeration and Gosper weights, written
 * to reproduce NumPy's results bit for bit:
 *   enumeration   geometry.py:161-171 (l1 outer, l2 >= l1, l3 from l2 or l2+1 by 2 to
 *                 min(l1+l2, l_max))
 *   multiplicity  geometry.py:114-123
 *   h2_gosper     geometry.py:97-110 (left-to-right products, 1.0/3.0, 1.0/6.0, pi**2)
 *   prefactor     geometry.py:140-141 (denom = 36*v1*v2*v3*sqrt(C1*C2*C3))
 *   zm            engine3d.py:133-134 (z * mult)
 * Build with -O2 -ffp-contract=off (no FMA contraction) — oracle/Makefile.
 */
#include <math.h>
#include <stdint.h>

static const double PI2 = 9.869604401089358; /* np.pi**2 */

int64_t or_row_len(int l1, int l2, int l_max) {
    int start = ((l1 + 2 * l2) % 2 == 0) ? l2 : l2 + 1;
    int stop = (l1 + l2 < l_max) ? l1 + l2 : l_max;
    return start > stop ? 0 : (stop - start) / 2 + 1;
}

int64_t or_domain_count(int l_min, int l_max) {
    int64_t n = 0;
    for (int l1 = l_min; l1 <= l_max; ++l1)
        for (int l2 = l1; l2 <= l_max; ++l2) n += or_row_len(l1, l2, l_max);
    return n;
}

/* triples with flat index in [begin, end) */
int64_t or_domain_triples(int l_min, int l_max, int64_t begin, int64_t end, int32_t* o1,
                          int32_t* o2, int32_t* o3) {
    int64_t t = 0, w = 0;
    for (int l1 = l_min; l1 <= l_max && t < end; ++l1) {
        for (int l2 = l1; l2 <= l_max && t < end; ++l2) {
            int64_t len = or_row_len(l1, l2, l_max);
            if (t + len <= begin) { t += len; continue; }
            int start = ((l1 + 2 * l2) % 2 == 0) ? l2 : l2 + 1;
            for (int64_t i = 0; i < len; ++i, ++t) {
                if (t < begin) continue;
                if (t >= end) break;
                o1[w] = l1; o2[w] = l2; o3[w] = start + 2 * (int)i; ++w;
            }
        }
    }
    return w;
}

int or_mult(int l1, int l2, int l3) {
    if (l1 == l3) return 1;
    if (l1 == l2 || l2 == l3) return 3;
    return 6;
}

double or_h2_gosper(int a, int b, int c) {
    double l1 = (double)a, l2 = (double)b, l3 = (double)c;
    double L = l1 + l2 + l3;
    double L1 = L - 2 * l1, L2 = L - 2 * l2, L3 = L - 2 * l3;
    double third = 1.0 / 3.0, sixth = 1.0 / 6.0;
    double num = (2 * l1 + 1) * (2 * l2 + 1) * (2 * l3 + 1) * (L + third);
    double den = (L + 1) * (L1 + third) * (L2 + third) * (L3 + third);
    double main_ = num / den;
    double root = sqrt((L1 + sixth) * (L2 + sixth) * (L3 + sixth) / (L + sixth));
    return main_ * root / (2.0 * PI2);
}

double or_zm(int l_min, int l1, int l2, int l3, const double* C, const double* v) {
    int i1 = l1 - l_min, i2 = l2 - l_min, i3 = l3 - l_min;
    double denom = 36.0 * v[i1] * v[i2] * v[i3] * sqrt(C[i1] * C[i2] * C[i3]);
    double z = or_h2_gosper(l1, l2, l3) / denom;
    return z * (double)or_mult(l1, l2, l3);
}

void or_weights(int l_min, int count, const int32_t* l1, const int32_t* l2, const int32_t* l3,
                const double* C, const double* v, double* zm) {
    for (int i = 0; i < count; ++i) zm[i] = or_zm(l_min, l1[i], l2[i], l3[i], C, v);
}
