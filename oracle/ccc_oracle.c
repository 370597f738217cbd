/*
 * oracle/ccc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU brute force of the CCC method of
 * PAPER.md (arXiv 1705.08213, Joubert et al.), used by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference leg.
 * Nothing in the product path (paper_1705_08213_b200/) may link, load or call
 * this file; it shares no code, header, table or constant with the CUDA path.
 *
 * Every function is a literal transcription of a definition of the paper:
 *
 *   element   v_{i,q} = (r1, r2) in S_2, S = {0,1}            (§2.1)
 *             stored as one byte code = 2*r1 + r2              (R-1)
 *   rho_{i,q}(a) = sum_r chi_a((v_{i,q})_r)
 *   S_i(a)  = sum_q rho_{i,q}(a),   f_i(a) = S_i(a) / (2 n_f)   (Eq.1)
 *   T_ij(a,b) = sum_q sum_{r in v_iq} sum_{r' in v_jq} [r=a][r'=b]
 *             -- the enumeration of all pairings of Fig.1,
 *                equal to sum_q rho_{i,q}(a) rho_{j,q}(b)       (Eq.2)
 *   f_ij = T_ij / (4 n_f)
 *   CCC_ij(a,b) = f_ij(a,b) (1 - g f_i(a)) (1 - g f_j(b))       (Eq.3)
 *   T_ijk(a,b,c): the 8 combinations of Fig.2      (Eq.5)
 *   f_ijk = T_ijk / (8 n_f)
 *   CCC_ijk(a,b,c) = f_ijk(a,b,c) prod (1 - g f(.))            (Eq.4)
 *
 * Unique results: pairs i<j, triples i<j<k, emitted in
 * lexicographic order, cells a-major (index 2a+b, 4a+2b+c).
 *
 * Tallies are accumulated in int64; CCC is evaluated in fp64 in the order the
 * equations are written.  OpenMP parallelises the outer record loop only.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <math.h>

/* (v_{i,q})_1 and (v_{i,q})_2 of the stored code (R-1). */
static int elem_r1(uint8_t code) { return (code >> 1) & 1; }
static int elem_r2(uint8_t code) { return code & 1; }

/* Eq.1 numerator: S_i(a) = sum_q rho_{i,q}(a), for a = 0,1.  S[i*2 + a]. */
void oracle_allele_sums(const uint8_t* codes, int64_t n_v, int64_t n_f, int64_t* S)
{
    for (int64_t i = 0; i < n_v; ++i) {
        int64_t s0 = 0, s1 = 0;
        for (int64_t q = 0; q < n_f; ++q) {
            uint8_t c = codes[i * n_f + q];
            int r[2] = {elem_r1(c), elem_r2(c)};
            for (int t = 0; t < 2; ++t) {          /* rho_{i,q}(a) = sum_r chi_a(r) */
                if (r[t] == 0) s0 += 1;
                if (r[t] == 1) s1 += 1;
            }
        }
        S[i * 2 + 0] = s0;
        S[i * 2 + 1] = s1;
    }
}

/* Fig.1 / Eq.2: the 2x2 tally of one pair, by enumerating the 4 pairings per field. */
static void tally2_one(const uint8_t* vi, const uint8_t* vj, int64_t n_f, int64_t T[4])
{
    T[0] = T[1] = T[2] = T[3] = 0;
    for (int64_t q = 0; q < n_f; ++q) {
        int ri[2] = {elem_r1(vi[q]), elem_r2(vi[q])};
        int rj[2] = {elem_r1(vj[q]), elem_r2(vj[q])};
        for (int s = 0; s < 2; ++s)
            for (int t = 0; t < 2; ++t)
                T[2 * ri[s] + rj[t]] += 1;          /* tuple (a,b) = (ri[s], rj[t]) */
    }
}

/* Fig.2 / Eq.5: the 2x2x2 tally of one triple, by enumerating the 8 combinations. */
static void tally3_one(const uint8_t* vi, const uint8_t* vj, const uint8_t* vk,
                       int64_t n_f, int64_t T[8])
{
    for (int c = 0; c < 8; ++c) T[c] = 0;
    for (int64_t q = 0; q < n_f; ++q) {
        int ri[2] = {elem_r1(vi[q]), elem_r2(vi[q])};
        int rj[2] = {elem_r1(vj[q]), elem_r2(vj[q])};
        int rk[2] = {elem_r1(vk[q]), elem_r2(vk[q])};
        for (int s = 0; s < 2; ++s)
            for (int t = 0; t < 2; ++t)
                for (int u = 0; u < 2; ++u)
                    T[4 * ri[s] + 2 * rj[t] + rk[u]] += 1;
    }
}

/* Eq.3 for one pair. */
static void ccc2_one(const int64_t T[4], const int64_t* Si, const int64_t* Sj,
                     int64_t n_f, double gamma, double out[4])
{
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            double f_ij = (double)T[2 * a + b] / (4.0 * (double)n_f);
            double f_ia = (double)Si[a] / (2.0 * (double)n_f);
            double f_jb = (double)Sj[b] / (2.0 * (double)n_f);
            out[2 * a + b] = f_ij * (1.0 - gamma * f_ia) * (1.0 - gamma * f_jb);
        }
}

/* Eq.4 for one triple. */
static void ccc3_one(const int64_t T[8], const int64_t* Si, const int64_t* Sj,
                     const int64_t* Sk, int64_t n_f, double gamma, double out[8])
{
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int c = 0; c < 2; ++c) {
                double f_ijk = (double)T[4 * a + 2 * b + c] / (8.0 * (double)n_f);
                double f_ia = (double)Si[a] / (2.0 * (double)n_f);
                double f_jb = (double)Sj[b] / (2.0 * (double)n_f);
                double f_kc = (double)Sk[c] / (2.0 * (double)n_f);
                out[4 * a + 2 * b + c] =
                    f_ijk * (1.0 - gamma * f_ia) * (1.0 - gamma * f_jb) * (1.0 - gamma * f_kc);
            }
}

/*
 * Tallies and CCC for an explicit list of pairs (idx[m][2], global vector ids).
 * S must come from oracle_allele_sums over the same codes.  ccc may be NULL.
 */
void oracle_pairs(const uint8_t* codes, int64_t n_v, int64_t n_f, const int64_t* S,
                  double gamma, const int64_t* idx, int64_t m, int64_t* T, double* ccc)
{
    (void)n_v;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = idx[2 * r], j = idx[2 * r + 1];
        tally2_one(codes + i * n_f, codes + j * n_f, n_f, T + 4 * r);
        if (ccc) ccc2_one(T + 4 * r, S + 2 * i, S + 2 * j, n_f, gamma, ccc + 4 * r);
    }
}

/* Same for an explicit list of triples (idx[m][3]). */
void oracle_triples(const uint8_t* codes, int64_t n_v, int64_t n_f, const int64_t* S,
                    double gamma, const int64_t* idx, int64_t m, int64_t* T, double* ccc)
{
    (void)n_v;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = idx[3 * r], j = idx[3 * r + 1], k = idx[3 * r + 2];
        tally3_one(codes + i * n_f, codes + j * n_f, codes + k * n_f, n_f, T + 8 * r);
        if (ccc)
            ccc3_one(T + 8 * r, S + 2 * i, S + 2 * j, S + 2 * k, n_f, gamma, ccc + 8 * r);
    }
}

/*
 * All unique pairs i<j in lexicographic order.  Record r of the
 * output is the r-th pair of the double loop below; T[C(n_v,2)][4], ccc likewise.
 */
void oracle_all_pairs(const uint8_t* codes, int64_t n_v, int64_t n_f, const int64_t* S,
                      double gamma, int64_t* T, double* ccc)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n_v; ++i) {
        /* records before row i: sum_{i' < i} (n_v - 1 - i') */
        int64_t r = 0;
        for (int64_t ii = 0; ii < i; ++ii) r += n_v - 1 - ii;
        for (int64_t j = i + 1; j < n_v; ++j, ++r) {
            tally2_one(codes + i * n_f, codes + j * n_f, n_f, T + 4 * r);
            if (ccc) ccc2_one(T + 4 * r, S + 2 * i, S + 2 * j, n_f, gamma, ccc + 4 * r);
        }
    }
}

/* All unique triples i<j<k in lexicographic order. */
void oracle_all_triples(const uint8_t* codes, int64_t n_v, int64_t n_f, const int64_t* S,
                        double gamma, int64_t* T, double* ccc)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n_v; ++i) {
        int64_t r = 0;                       /* records before pivot row i, counted */
        for (int64_t ii = 0; ii < i; ++ii)
            for (int64_t jj = ii + 1; jj < n_v; ++jj) r += n_v - 1 - jj;
        for (int64_t j = i + 1; j < n_v; ++j)
            for (int64_t k = j + 1; k < n_v; ++k, ++r) {
                tally3_one(codes + i * n_f, codes + j * n_f, codes + k * n_f, n_f, T + 8 * r);
                if (ccc)
                    ccc3_one(T + 8 * r, S + 2 * i, S + 2 * j, S + 2 * k, n_f, gamma,
                             ccc + 8 * r);
            }
    }
}

/*
 * ---- Sparse (missing-data) mode, §7 item 1 -------------------
 * "the value (1,0) can be set aside as a marker to denote a missing entry ... skipping
 * calculations for missing entries".  Reading A-17:
 *   present_{i,q} = [v_{i,q} != (1,0)],  c_i = sum_q present_{i,q}
 *   S_i(a)  = sum over present q of rho_{i,q}(a),   f_i(a) = S_i(a) / (2 c_i)
 *   T_ij(a,b) = the Fig.1 enumeration over the fields where BOTH entries are present,
 *   c_ij = that number of fields,  f_ij = T_ij / (4 c_ij)
 *   CCC_ij(a,b) = f_ij(a,b) (1 - g f_i(a)) (1 - g f_j(b))          (Eq.3 with these)
 * Degenerate cases: c_ij = 0 -> T = 0 and CCC = 0; c_i = 0 -> f_i(a) = 0.
 */
static int elem_missing(uint8_t code) { return elem_r1(code) == 1 && elem_r2(code) == 0; }

/* S[i*2 + a] over present entries, cnt[i] = c_i. */
void oracle_sparse_sums(const uint8_t* codes, int64_t n_v, int64_t n_f, int64_t* S,
                        int64_t* cnt)
{
    for (int64_t i = 0; i < n_v; ++i) {
        int64_t s0 = 0, s1 = 0, c = 0;
        for (int64_t q = 0; q < n_f; ++q) {
            uint8_t e = codes[i * n_f + q];
            if (elem_missing(e)) continue;
            c += 1;
            int r[2] = {elem_r1(e), elem_r2(e)};
            for (int t = 0; t < 2; ++t) {
                if (r[t] == 0) s0 += 1;
                if (r[t] == 1) s1 += 1;
            }
        }
        S[i * 2 + 0] = s0;
        S[i * 2 + 1] = s1;
        cnt[i] = c;
    }
}

static void tally2_sparse_one(const uint8_t* vi, const uint8_t* vj, int64_t n_f, int64_t T[4],
                              int64_t* c_ij)
{
    T[0] = T[1] = T[2] = T[3] = 0;
    *c_ij = 0;
    for (int64_t q = 0; q < n_f; ++q) {
        if (elem_missing(vi[q]) || elem_missing(vj[q])) continue;   /* skipped field */
        *c_ij += 1;
        int ri[2] = {elem_r1(vi[q]), elem_r2(vi[q])};
        int rj[2] = {elem_r1(vj[q]), elem_r2(vj[q])};
        for (int s = 0; s < 2; ++s)
            for (int t = 0; t < 2; ++t)
                T[2 * ri[s] + rj[t]] += 1;
    }
}

static void ccc2_sparse_one(const int64_t T[4], const int64_t* Si, const int64_t* Sj,
                            int64_t c_i, int64_t c_j, int64_t c_ij, double gamma, double out[4])
{
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            if (c_ij == 0) {
                out[2 * a + b] = 0.0;
                continue;
            }
            double f_ij = (double)T[2 * a + b] / (4.0 * (double)c_ij);
            double f_ia = c_i ? (double)Si[a] / (2.0 * (double)c_i) : 0.0;
            double f_jb = c_j ? (double)Sj[b] / (2.0 * (double)c_j) : 0.0;
            out[2 * a + b] = f_ij * (1.0 - gamma * f_ia) * (1.0 - gamma * f_jb);
        }
}

/* Sparse tallies, CCC and c_ij for an explicit pair list idx[m][2]; S, cnt from
 * oracle_sparse_sums.  ccc / cij may be NULL. */
void oracle_sparse_pairs(const uint8_t* codes, int64_t n_v, int64_t n_f, const int64_t* S,
                         const int64_t* cnt, double gamma, const int64_t* idx, int64_t m,
                         int64_t* T, double* ccc, int64_t* cij)
{
    (void)n_v;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < m; ++r) {
        int64_t i = idx[2 * r], j = idx[2 * r + 1], c;
        tally2_sparse_one(codes + i * n_f, codes + j * n_f, n_f, T + 4 * r, &c);
        if (cij) cij[r] = c;
        if (ccc)
            ccc2_sparse_one(T + 4 * r, S + 2 * i, S + 2 * j, cnt[i], cnt[j], c, gamma,
                            ccc + 4 * r);
    }
}

/*
 * ---- Sparse (missing-data) mode, 3-way: the same reading A-17 for triples,
 * SPEC's "per-triple valid counts in the f_{i,j,k} divisor and per-vector valid counts
 * for f_i":
 *   T_ijk(a,b,c) = the Fig.2 enumeration over the fields where ALL THREE are present,
 *   c_ijk = that number of fields,  f_ijk = T_ijk / (8 c_ijk)
 *   CCC_ijk(a,b,c) = f_ijk(a,b,c) (1 - g f_i(a)) (1 - g f_j(b)) (1 - g f_k(c))   (Eq.4)
 *   with f_i(a) = S_i(a) / (2 c_i) over vector i's present entries (0 if c_i = 0);
 *   c_ijk = 0 -> T = 0 and CCC = 0.
 */
static void tally3_sparse_one(const uint8_t* vi, const uint8_t* vj, const uint8_t* vk, int64_t n_f,
                              int64_t T[8], int64_t* c_ijk)
{
    for (int t = 0; t < 8; ++t) T[t] = 0;
    *c_ijk = 0;
    for (int64_t q = 0; q < n_f; ++q) {
        if (elem_missing(vi[q]) || elem_missing(vj[q]) || elem_missing(vk[q])) continue;
        *c_ijk += 1;
        int ri[2] = {elem_r1(vi[q]), elem_r2(vi[q])};
        int rj[2] = {elem_r1(vj[q]), elem_r2(vj[q])};
        int rk[2] = {elem_r1(vk[q]), elem_r2(vk[q])};
        for (int s = 0; s < 2; ++s)
            for (int t = 0; t < 2; ++t)
                for (int u = 0; u < 2; ++u)
                    T[4 * ri[s] + 2 * rj[t] + rk[u]] += 1;
    }
}

/* Sparse 3-way tallies, CCC and c_ijk for an explicit triple list idx[m][3]; S, cnt from
 * oracle_sparse_sums.  ccc / cijk may be NULL. */
void oracle_sparse_triples(const uint8_t* codes, int64_t n_v, int64_t n_f, const int64_t* S,
                           const int64_t* cnt, double gamma, const int64_t* idx, int64_t m,
                           int64_t* T, double* ccc, int64_t* cijk)
{
    (void)n_v;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < m; ++r) {
        const int64_t ix[3] = {idx[3 * r], idx[3 * r + 1], idx[3 * r + 2]};
        int64_t c;
        tally3_sparse_one(codes + ix[0] * n_f, codes + ix[1] * n_f, codes + ix[2] * n_f, n_f,
                          T + 8 * r, &c);
        if (cijk) cijk[r] = c;
        if (!ccc) continue;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int d = 0; d < 2; ++d) {
                    const int cell = 4 * a + 2 * b + d;
                    if (c == 0) {
                        ccc[8 * r + cell] = 0.0;
                        continue;
                    }
                    const int al[3] = {a, b, d};
                    double f_ijk = (double)T[8 * r + cell] / (8.0 * (double)c);
                    double v = f_ijk;
                    for (int t = 0; t < 3; ++t) {
                        const int64_t x = ix[t];
                        double f = cnt[x] ? (double)S[2 * x + al[t]] / (2.0 * (double)cnt[x]) : 0.0;
                        v *= (1.0 - gamma * f);
                    }
                    ccc[8 * r + cell] = v;
                }
    }
}

/*
 * ---- Planted type-2 data: the closed form (§5: "randomized placement
 * of entries specifically chosen so that the correctness of every result value can be
 * verified analytically").
 *
 * Before the column permutation, vector i holds (1,1) on the fields [0, L_i), a
 * heterozygote on [L_i, E_i) with E_i = L_i + H_i, and (0,0) on [E_i, n_f).  One column
 * permutation shared by all vectors reorders the terms of every sum over q and changes
 * none of them.  So rho_{i,q}(1) = [q < L_i] + [q < E_i] and rho_{i,q}(0) = 2 - rho_{i,q}(1)
 * are constant between consecutive breakpoints {0, L, E, n_f} of the vectors
 * involved, and every sum over q of Eq.1, Eq.2 and Eq.5 is a sum over those pieces of
 * (piece width) x (the product of the rho's on the piece).  CCC then follows Eq.3 / Eq.4
 * exactly as for the brute force above (ccc2_one / ccc3_one).
 * Pinned (tests/test_oracle.py) record for record against the brute force on the
 * generated planted codes and against the Python interval form oracle.planted_tally2/3.
 */
static int64_t planted_rho(int64_t L, int64_t E, int64_t q, int a)
{
    int64_t one = (q < L) + (q < E);         /* allele-1 count of field q */
    return a ? one : 2 - one;
}

static void sort_small(int64_t* x, int n)
{
    for (int p = 1; p < n; ++p) {
        int64_t v = x[p];
        int t = p - 1;
        while (t >= 0 && x[t] > v) { x[t + 1] = x[t]; --t; }
        x[t + 1] = v;
    }
}

/* Eq.1 numerators S_i(a) of every planted vector: S[i*2 + a]. */
void oracle_planted_sums(const int64_t* L, const int64_t* H, int64_t n_v, int64_t n_f, int64_t* S)
{
    for (int64_t i = 0; i < n_v; ++i) {
        int64_t b[4] = {0, L[i], L[i] + H[i], n_f};
        sort_small(b, 4);
        S[2 * i] = S[2 * i + 1] = 0;
        for (int p = 0; p < 3; ++p) {
            int64_t w = b[p + 1] - b[p];
            if (w <= 0) continue;
            for (int a = 0; a < 2; ++a) S[2 * i + a] += w * planted_rho(L[i], L[i] + H[i], b[p], a);
        }
    }
}

/* Eq.2 tally of the planted pair (i, j), piece by piece. */
static void planted_tally2_one(const int64_t* L, const int64_t* H, int64_t n_f, int64_t i,
                               int64_t j, int64_t T[4])
{
    const int64_t Ei = L[i] + H[i], Ej = L[j] + H[j];
    int64_t b[6] = {0, L[i], Ei, L[j], Ej, n_f};
    sort_small(b, 6);
    T[0] = T[1] = T[2] = T[3] = 0;
    for (int p = 0; p < 5; ++p) {
        int64_t w = b[p + 1] - b[p];
        if (w <= 0) continue;
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 2; ++c)
                T[2 * a + c] += w * planted_rho(L[i], Ei, b[p], a) * planted_rho(L[j], Ej, b[p], c);
    }
}

/* Eq.5 tally of the planted triple (i, j, k), piece by piece. */
static void planted_tally3_one(const int64_t* L, const int64_t* H, int64_t n_f, int64_t i,
                               int64_t j, int64_t k, int64_t T[8])
{
    const int64_t Ei = L[i] + H[i], Ej = L[j] + H[j], Ek = L[k] + H[k];
    int64_t b[8] = {0, L[i], Ei, L[j], Ej, L[k], Ek, n_f};
    sort_small(b, 8);
    for (int t = 0; t < 8; ++t) T[t] = 0;
    for (int p = 0; p < 7; ++p) {
        int64_t w = b[p + 1] - b[p];
        if (w <= 0) continue;
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 2; ++c)
                for (int d = 0; d < 2; ++d)
                    T[4 * a + 2 * c + d] += w * planted_rho(L[i], Ei, b[p], a) *
                                            planted_rho(L[j], Ej, b[p], c) *
                                            planted_rho(L[k], Ek, b[p], d);
    }
}

/* Number of unique pairs (i', j') with i' < i: rows 0..i-1 of the lexicographic order. */
static int64_t pairs_before_row(int64_t n_v, int64_t i)
{
    return i * (2 * n_v - i - 1) / 2;        /* sum_{i' < i} (n_v - 1 - i') */
}

/* Records of the planted pairs [rec0, rec0 + nrec) of the lexicographic order:
 * T[nrec][4] int64 and (if ccc) CCC fp64 by Eq.3 from the closed-form S. */
void oracle_planted_pairs(const int64_t* L, const int64_t* H, int64_t n_v, int64_t n_f,
                          double gamma, int64_t rec0, int64_t nrec, int64_t* T, double* ccc)
{
    int64_t* Sv = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(n_v ? n_v : 1));
    oracle_planted_sums(L, H, n_v, n_f, Sv);
    int64_t i0 = 0;
    while (i0 < n_v && pairs_before_row(n_v, i0 + 1) <= rec0) ++i0;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = i0; i < n_v; ++i) {
        int64_t r = pairs_before_row(n_v, i) - rec0;          /* record of (i, i+1) */
        if (r >= nrec) continue;
        for (int64_t j = i + 1; j < n_v; ++j, ++r) {
            if (r < 0 || r >= nrec) continue;
            planted_tally2_one(L, H, n_f, i, j, T + 4 * r);
            if (ccc) ccc2_one(T + 4 * r, Sv + 2 * i, Sv + 2 * j, n_f, gamma, ccc + 4 * r);
        }
    }
    free(Sv);
}

/* Same for triples [rec0, rec0 + nrec) of the lexicographic order. */
void oracle_planted_triples(const int64_t* L, const int64_t* H, int64_t n_v, int64_t n_f,
                            double gamma, int64_t rec0, int64_t nrec, int64_t* T, double* ccc)
{
    int64_t* Sv = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(n_v ? n_v : 1));
    oracle_planted_sums(L, H, n_v, n_f, Sv);
    for (int64_t i = 0, base = 0; i < n_v; base += (n_v - 1 - i) * (n_v - 2 - i) / 2, ++i) {
        if (base >= rec0 + nrec) break;
        if (base + (n_v - 1 - i) * (n_v - 2 - i) / 2 <= rec0) continue;
        #pragma omp parallel for schedule(dynamic, 4)
        for (int64_t j = i + 1; j < n_v; ++j) {
            /* records of row i before (i, j, j+1): sum_{j' = i+1}^{j-1} (n_v - 1 - j') */
            int64_t r = base - rec0;
            for (int64_t jj = i + 1; jj < j; ++jj) r += n_v - 1 - jj;
            for (int64_t k = j + 1; k < n_v; ++k, ++r) {
                if (r < 0 || r >= nrec) continue;
                planted_tally3_one(L, H, n_f, i, j, k, T + 8 * r);
                if (ccc)
                    ccc3_one(T + 8 * r, Sv + 2 * i, Sv + 2 * j, Sv + 2 * k, n_f, gamma,
                             ccc + 8 * r);
            }
        }
    }
    free(Sv);
}

/*
 * Full-size checker (test infrastructure): compare records a CALLER copied back from the
 * device -- tallies uint32 [nrec][cells], CCC fp64 or fp32 [nrec][cells] (ccc_bytes 8 / 4,
 * 0 = none) -- for the records [rec0, rec0 + nrec) of the lexicographic order against the
 * planted closed form above, one record at a time (nothing expected is stored).
 * Bars: tallies bit-exact; CCC |x - y| <= rtol |y| and x == 0 exactly where
 * y == 0.  res[0] = records whose tallies differ, res[1] = records with a CCC cell outside
 * the bar, res[2] = the first bad record (-1 if none); *max_rel = the largest relative CCC
 * error seen.
 */
static void check_cells(const int64_t* Te, const double* Ce, int cells, const uint32_t* Tg,
                        const void* Cg, int ccc_bytes, int64_t r, double rtol,
                        int64_t* bad_t, int64_t* bad_c, int64_t* first, double* mrel)
{
    int tb = 0, cb = 0;
    if (Tg)
        for (int c = 0; c < cells; ++c)
            if ((int64_t)Tg[(size_t)r * cells + c] != Te[c]) tb = 1;
    if (ccc_bytes)
        for (int c = 0; c < cells; ++c) {
            double g = ccc_bytes == 8 ? ((const double*)Cg)[(size_t)r * cells + c]
                                      : (double)((const float*)Cg)[(size_t)r * cells + c];
            double y = Ce[c];
            if (y == 0.0) {
                if (g != 0.0) cb = 1;
                continue;
            }
            double rel = fabs(g - y) / fabs(y);
            if (!(rel <= rtol)) cb = 1;           /* NaN fails too */
            if (rel > *mrel || rel != rel) *mrel = rel != rel ? INFINITY : rel;
        }
    if (tb) ++*bad_t;
    if (cb) ++*bad_c;
    if ((tb || cb) && (*first < 0 || r < *first)) *first = r;
}

void oracle_planted_check2(const int64_t* L, const int64_t* H, int64_t n_v, int64_t n_f,
                           double gamma, int64_t rec0, int64_t nrec, const uint32_t* Tg,
                           const void* Cg, int ccc_bytes, double rtol, int64_t* res,
                           double* max_rel)
{
    int64_t* Sv = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(n_v ? n_v : 1));
    oracle_planted_sums(L, H, n_v, n_f, Sv);
    int64_t bad_t = 0, bad_c = 0, first = -1;
    double mrel = 0.0;
    int64_t i0 = 0;
    while (i0 < n_v && pairs_before_row(n_v, i0 + 1) <= rec0) ++i0;
    #pragma omp parallel
    {
        int64_t bt = 0, bc = 0, fb = -1;
        double mr = 0.0;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = i0; i < n_v; ++i) {
            int64_t r = pairs_before_row(n_v, i) - rec0;
            if (r >= nrec) continue;
            for (int64_t j = i + 1; j < n_v; ++j, ++r) {
                if (r < 0 || r >= nrec) continue;
                int64_t Te[4];
                double Ce[4];
                planted_tally2_one(L, H, n_f, i, j, Te);
                ccc2_one(Te, Sv + 2 * i, Sv + 2 * j, n_f, gamma, Ce);
                check_cells(Te, Ce, 4, Tg, Cg, ccc_bytes, r, rtol, &bt, &bc, &fb, &mr);
            }
        }
        #pragma omp critical
        {
            bad_t += bt;
            bad_c += bc;
            if (fb >= 0 && (first < 0 || fb < first)) first = fb;
            if (mr > mrel) mrel = mr;
        }
    }
    res[0] = bad_t;
    res[1] = bad_c;
    res[2] = first;
    *max_rel = mrel;
    free(Sv);
}

/*
 * The 3-way checker visits ~1e10 triples at C4, so it evaluates the same closed form with
 * the work that does not depend on k hoisted out of the k loop -- the same arithmetic:
 *   - the pieces of [0, n_f) on which rho_i and rho_j are constant and the products
 *     rho_i(a) rho_j(b) on them (planted_tally3_one's breakpoints of i and j);
 *   - k splits a piece [x0, x0 + w) at L_k and E_k, and sum_{q in piece} rho_k(1) =
 *     |piece & [0, L_k)| + |piece & [0, E_k)|, sum rho_k(0) = 2w - that;
 *   - the per-vector factors (1 - g f_v(a)) of Eq.4, computed as in ccc3_one and
 *     multiplied in ccc3_one's order, so CCC is bit-identical to it.
 * tests/test_oracle.py pins the checker at rtol = 0 against oracle_planted_triples.
 */
typedef struct {
    int np;
    int64_t x0[5], w[5], P[5][4];            /* P[p][2a+b] = rho_i(a) rho_j(b) on piece p */
} pair_pieces;

static void planted_pieces(const int64_t* L, const int64_t* H, int64_t n_f, int64_t i,
                           int64_t j, pair_pieces* pp)
{
    const int64_t Ei = L[i] + H[i], Ej = L[j] + H[j];
    int64_t b[6] = {0, L[i], Ei, L[j], Ej, n_f};
    sort_small(b, 6);
    pp->np = 0;
    for (int p = 0; p < 5; ++p) {
        int64_t w = b[p + 1] - b[p];
        if (w <= 0) continue;
        int n = pp->np++;
        pp->x0[n] = b[p];
        pp->w[n] = w;
        for (int a = 0; a < 2; ++a)
            for (int c = 0; c < 2; ++c)
                pp->P[n][2 * a + c] = planted_rho(L[i], Ei, b[p], a) * planted_rho(L[j], Ej, b[p], c);
    }
}

static int64_t clamp64(int64_t x, int64_t lo, int64_t hi) { return x < lo ? lo : x > hi ? hi : x; }

static void planted_tally3_k(const pair_pieces* pp, int64_t Lk, int64_t Ek, int64_t T[8])
{
    for (int t = 0; t < 8; ++t) T[t] = 0;
    for (int n = 0; n < pp->np; ++n) {
        int64_t x0 = pp->x0[n], w = pp->w[n];
        int64_t one = clamp64(Lk - x0, 0, w) + clamp64(Ek - x0, 0, w);
        int64_t zero = 2 * w - one;
        for (int ab = 0; ab < 4; ++ab) {
            T[2 * ab + 0] += pp->P[n][ab] * zero;
            T[2 * ab + 1] += pp->P[n][ab] * one;
        }
    }
}

void oracle_planted_check3(const int64_t* L, const int64_t* H, int64_t n_v, int64_t n_f,
                           double gamma, int64_t rec0, int64_t nrec, const uint32_t* Tg,
                           const void* Cg, int ccc_bytes, double rtol, int64_t* res,
                           double* max_rel)
{
    int64_t* Sv = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(n_v ? n_v : 1));
    double* Wv = (double*)malloc(sizeof(double) * 2 * (size_t)(n_v ? n_v : 1));
    oracle_planted_sums(L, H, n_v, n_f, Sv);
    for (int64_t v = 0; v < 2 * n_v; ++v)                   /* 1 - g f_v(a), as ccc3_one */
        Wv[v] = 1.0 - gamma * ((double)Sv[v] / (2.0 * (double)n_f));
    int64_t bad_t = 0, bad_c = 0, first = -1;
    double mrel = 0.0;
    for (int64_t i = 0, base = 0; i < n_v; base += (n_v - 1 - i) * (n_v - 2 - i) / 2, ++i) {
        if (base >= rec0 + nrec) break;
        if (base + (n_v - 1 - i) * (n_v - 2 - i) / 2 <= rec0) continue;
        #pragma omp parallel
        {
            int64_t bt = 0, bc = 0, fb = -1;
            double mr = 0.0;
            #pragma omp for schedule(dynamic, 4)
            for (int64_t j = i + 1; j < n_v; ++j) {
                int64_t r = base - rec0;
                for (int64_t jj = i + 1; jj < j; ++jj) r += n_v - 1 - jj;
                if (r >= nrec || r + (n_v - 1 - j) <= 0) continue;
                pair_pieces pp;
                planted_pieces(L, H, n_f, i, j, &pp);
                for (int64_t k = j + 1; k < n_v; ++k, ++r) {
                    if (r < 0 || r >= nrec) continue;
                    int64_t Te[8];
                    double Ce[8];
                    planted_tally3_k(&pp, L[k], L[k] + H[k], Te);
                    for (int a = 0; a < 2; ++a)
                        for (int b = 0; b < 2; ++b)
                            for (int c = 0; c < 2; ++c) {
                                int cell = 4 * a + 2 * b + c;
                                double f_ijk = (double)Te[cell] / (8.0 * (double)n_f);
                                Ce[cell] = f_ijk * Wv[2 * i + a] * Wv[2 * j + b] * Wv[2 * k + c];
                            }
                    check_cells(Te, Ce, 8, Tg, Cg, ccc_bytes, r, rtol, &bt, &bc, &fb, &mr);
                }
            }
            #pragma omp critical
            {
                bad_t += bt;
                bad_c += bc;
                if (fb >= 0 && (first < 0 || fb < first)) first = fb;
                if (mr > mrel) mrel = mr;
            }
        }
    }
    res[0] = bad_t;
    res[1] = bad_c;
    res[2] = first;
    *max_rel = mrel;
    free(Sv);
    free(Wv);
}
