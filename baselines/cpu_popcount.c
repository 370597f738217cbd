/* cpu_popcount.c -- SURVEY §8(f) f4(iii): an optimized bit-packed CPU version of the 2-way
 * tally, the paper's "optimized CPU version" comparison line.
 *
 * A REPORTED BASELINE, not the product and not the oracle: bench.py times it on the host
 * cores beside the oracle; the CUDA path never calls it.  Its tests compare it with the
 * oracle (tests/test_cpu_popcount.py).
 *
 * Input: the packed rows of ccc_pack (2 bits per genotype, code = (r1 << 1) | r2, LSB
 * first, rows of ceil(n_f/64)*16 bytes, zero padding).  Per 64-bit word pair (32 codes)
 *   sum n_i n_j = popcount(x & y) + popcount(((x >> 1) & L & y) | ((x << 1) & y & H)),
 * n = r1 + r2, L = 0x5555..., H = 0xAAAA... (same identity as the GPU popcount kernel),
 * then Eq.2-3: T11 = G, T10 = 2s_i - G, T01 = 2s_j - G, T00 = 4n_f - 2s_i - 2s_j + G,
 * CCC(a,b) = T(a,b)/(4n_f) w_i(a) w_j(b), w(a) = 1 - gamma f(a) (Eq.1).
 * Blocked over j (64 rows) for cache reuse, OpenMP over i. */
#include <stdint.h>
#include <stddef.h>

#define L64 0x5555555555555555ull
#define H64 0xAAAAAAAAAAAAAAAAull

static inline int64_t pair_index(int64_t n_v, int64_t i, int64_t j) {
    return i * (2 * n_v - i - 1) / 2 + (j - i - 1);
}

/* Tallies [C(n_v,2)][4] and CCC [..][4] (either may be NULL) for every pair (i, j), i in
 * [i_lo, i_hi), j > i, at the global pair index minus the index of (i_lo, i_lo + 1). */
void cpu_popcount_2way(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma,
                       int64_t i_lo, int64_t i_hi, uint32_t* tallies, double* ccc) {
    const int64_t wpr = (n_f + 63) / 64 * 2;   /* 64-bit words per row */
    const uint64_t* P = (const uint64_t*)packed;
    const int64_t base = (i_lo < n_v - 1) ? pair_index(n_v, i_lo, i_lo + 1) : 0;
    const double inv4 = 1.0 / (4.0 * (double)n_f), two_nf = 2.0 * (double)n_f;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = i_lo; i < i_hi; ++i) {
        const uint64_t* x = P + i * wpr;
        uint32_t si = 0;
        for (int64_t w = 0; w < wpr; ++w) si += (uint32_t)__builtin_popcountll(x[w]);
        const double wi0 = 1.0 - gamma * ((two_nf - si) / two_nf), wi1 = 1.0 - gamma * (si / two_nf);
        for (int64_t j0 = i + 1; j0 < n_v; j0 += 64) {
            const int64_t j1 = j0 + 64 < n_v ? j0 + 64 : n_v;
            uint32_t g[64] = {0};
            for (int64_t w = 0; w < wpr; ++w) {
                const uint64_t a = x[w], as = (a >> 1) & L64, al = a << 1;
                for (int64_t j = j0; j < j1; ++j) {
                    const uint64_t y = P[j * wpr + w];
                    g[j - j0] += (uint32_t)(__builtin_popcountll(a & y) +
                                            __builtin_popcountll((as & y) | (al & y & H64)));
                }
            }
            for (int64_t j = j0; j < j1; ++j) {
                const uint64_t* yr = P + j * wpr;
                uint32_t sj = 0;
                for (int64_t w = 0; w < wpr; ++w) sj += (uint32_t)__builtin_popcountll(yr[w]);
                const uint32_t G = g[j - j0];
                const uint32_t t11 = G, t10 = 2u * si - G, t01 = 2u * sj - G;
                const uint32_t t00 = 4u * (uint32_t)n_f - 2u * si - 2u * sj + G;
                const int64_t r = pair_index(n_v, i, j) - base;
                if (tallies) {
                    tallies[4 * r + 0] = t00;
                    tallies[4 * r + 1] = t01;
                    tallies[4 * r + 2] = t10;
                    tallies[4 * r + 3] = t11;
                }
                if (ccc) {
                    const double wj0 = 1.0 - gamma * ((two_nf - sj) / two_nf), wj1 = 1.0 - gamma * (sj / two_nf);
                    ccc[4 * r + 0] = (double)t00 * inv4 * wi0 * wj0;
                    ccc[4 * r + 1] = (double)t01 * inv4 * wi0 * wj1;
                    ccc[4 * r + 2] = (double)t10 * inv4 * wi1 * wj0;
                    ccc[4 * r + 3] = (double)t11 * inv4 * wi1 * wj1;
                }
            }
        }
    }
}
