// common.cuh -- structures shared by the CCC kernels and their host launchers.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

namespace ccc {

constexpr int kBM = 128;        // tile rows   (UMMA M, one TMEM lane per row)
constexpr int kBN = 256;        // tile cols   (UMMA N, TMEM columns per accumulator)
constexpr int kBK = 128;        // K bytes per pipeline stage (one 128-B swizzle atom)
constexpr int kUMMA_K = 32;     // K of one kind::i8 tcgen05.mma

// Record digest for the order-independent checksum (R-9).
constexpr uint64_t kCkSeed = 0x243F6A8885A308D3ull;
constexpr uint64_t kCkHi = 0x13198A2E03707344ull;

// 2-way tile space: rows [a_lo, a_lo + nA) of block A against cols [0, nB) of block B,
// tiles of bm x kBN (bm = 128 for one CTA, 256 for a CTA pair).
// diag: A and B are one block and only local pairs i < j are wanted.
// Tiles are visited in super-tile order (2048 x 2048 elements, row-major over super
// tiles, row-major inside) so that the ~148 concurrently active tiles share few A / B
// panels in L2.
struct TriSched {
    int64_t a_lo, nA, nB, b_lo;   // rows [a_lo, a_lo+nA); cols [b_lo, b_lo+nB) (b_lo = 0 if diag)
    int32_t diag, bm_rows, sup_m, sup_n, nbm, nbn, SP, SQ;
    // cursor
    int32_t P, Q, cnt;
    int64_t base;

    __host__ __device__ void init(int64_t a_lo_, int64_t nA_, int64_t nB_, int diag_,
                                  int32_t bm_rows_ = kBM, int32_t sup_rows = 2048,
                                  int32_t sup_cols = 2048) {
        a_lo = a_lo_;
        nA = nA_;
        nB = nB_;
        b_lo = 0;
        diag = diag_;
        bm_rows = bm_rows_;
        sup_m = sup_rows / bm_rows > 0 ? sup_rows / bm_rows : 1;
        sup_n = sup_cols / kBN > 0 ? sup_cols / kBN : 1;
        nbm = (int32_t)((nA + bm_rows - 1) / bm_rows);
        nbn = (int32_t)((nB + kBN - 1) / kBN);
        SP = (nbm + sup_m - 1) / sup_m;
        SQ = (nbn + sup_n - 1) / sup_n;
        P = 0;
        Q = 0;
        base = 0;
        cnt = (SP > 0 && SQ > 0) ? super_count(0, 0) : 0;
    }
    // first valid column tile for row tile bm (diag), or 0 (rect); nbn if none.
    __host__ __device__ int32_t bn_first(int32_t bm) const {
        if (!diag) return 0;
        int64_t i_min = a_lo + (int64_t)bm * bm_rows;
        if (i_min >= nB - 1) return nbn;
        // need bn*kBN + kBN - 1 > i_min  <=>  bn >= floor((i_min + 1) / kBN)
        return (int32_t)((i_min + 1) / kBN);
    }
    __host__ __device__ int32_t row_count(int32_t bm, int32_t Qs) const {
        int32_t lo = Qs * sup_n, hi = lo + sup_n;
        if (hi > nbn) hi = nbn;
        int32_t f = bn_first(bm);
        if (f > lo) lo = f;
        return hi > lo ? hi - lo : 0;
    }
    __host__ __device__ int32_t super_count(int32_t Ps, int32_t Qs) const {
        int32_t r0 = Ps * sup_m, r1 = r0 + sup_m, c = 0;
        if (r1 > nbm) r1 = nbm;
        for (int32_t bm = r0; bm < r1; ++bm) c += row_count(bm, Qs);
        return c;
    }
    // Map the (monotonically increasing) linear tile index t -> (bm, bn).
    __host__ __device__ bool get(int64_t t, int32_t& bm, int32_t& bn) {
        while (t >= base + cnt) {
            base += cnt;
            if (++Q == SQ) {
                Q = 0;
                if (++P == SP) { cnt = 0; return false; }
            }
            cnt = super_count(P, Q);
        }
        int64_t local = t - base;
        int32_t r0 = P * sup_m, r1 = r0 + sup_m;
        if (r1 > nbm) r1 = nbm;
        for (int32_t r = r0; r < r1; ++r) {
            int32_t c = row_count(r, Q);
            if (local < c) {
                int32_t lo = Q * sup_n, f = bn_first(r);
                bm = r;
                bn = (f > lo ? f : lo) + (int32_t)local;
                return true;
            }
            local -= c;
        }
        return false;  // unreachable
    }
    __host__ int64_t total() {
        int64_t s = 0;
        for (int32_t p = 0; p < SP; ++p)
            for (int32_t q = 0; q < SQ; ++q) s += super_count(p, q);
        return s;
    }
};

// Kernel arguments of the fused 2-way tally GEMM (KB-2W).
// Threshold-compacted output: instead of the dense record
// arrays, every record whose largest CCC cell exceeds `thr` is appended at
// slot = atomicAdd(count, 1) (warp-aggregated): keys[slot] = global index key,
// tallies[slot][cells], ccc[slot][cells].  Slots >= cap are counted but not stored.
struct Compact {
    double thr;
    int64_t cap;
    unsigned long long* keys;
    unsigned long long* count;
};

// Next free slot of a compacted output: one atomic per group of converged threads.
__device__ __forceinline__ unsigned long long compact_slot(unsigned long long* count) {
    namespace cg = cooperative_groups;
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(count, (unsigned long long)g.size());
    return g.shfl(base, 0) + g.thread_rank();
}

struct Tally2Args {
    int64_t a_lo, nA, nB;      // A rows [a_lo, a_lo+nA) (local), B rows [0, nB)
    int64_t a_row0, b_row0;    // global index of local row 0 of A / B (checksum)
    int32_t diag;
    int32_t n_f;
    int32_t k_blocks;          // K_pad / kBK
    int32_t out_flags;
    const int32_t* s_a;
    const int32_t* s_b;
    const double* w_a;         // [rows][2]
    const double* w_b;
    uint32_t* tallies;         // [records][4]
    void* ccc;                 // [records][4] double or float
    unsigned long long* checksum;  // [2]
    int32_t* g_out;            // optional raw G
    int64_t ldg;
    int64_t rec_row_base;      // diag: record index of row a_lo's first pair
    int32_t sup_rows, sup_cols;  // super-tile shape (elements) of the tile raster
    int32_t k_alternate;         // odd waves of tiles walk K backwards (L2 reuse across waves)
    int32_t exact23;             // gamma == 2/3: CCC = double(T*U_i(a)) * (U_j(b)/D), D = 36 n_f^3
    double inv_d;                // 1 / (36 n_f^3)
    Compact cmp;                 // used when compact != 0
    int32_t compact;
    // sparse mode (f1): a_lo / nA / nB above are in rows of the group-interleaved X;
    // the records cover vectors [v_lo, v_hi) of A (local) x [0, nBv) of B
    int32_t sparse;
    int64_t v_lo, v_hi, nBv;
    const int32_t* c_a;          // present-entry counts c_i
    const int32_t* c_b;
    unsigned long long* trace; // optional per-tile %globaltimer trace (diagnostics)
    // f3 field split: schedule range and partial-G export (no records are written)
    int64_t t_lo, t_hi;          // tiles [t_lo, t_hi) of the schedule; t_hi = 0: all
    int32_t* const* xp_ptrs;     // [xp_world] owner slot buffers (device-visible), or NULL
    int32_t xp_rank, xp_world;   // this field slice; number of slices (= owners)
};

// f3 field split: the 2-way block whose tiles are exported / finished (the geometry of
// ccc_2way_block: rows [a_lo, a_lo + nA) of block A against the nB rows of block B; diag:
// A and B are one block and only i < j; a_row0 / b_row0 global index of local row 0).
struct FsGeom {
    int64_t a_lo, nA, nB, a_row0, b_row0;
    int32_t diag, pad_;
};

// One vector block as seen by the 3-way kernel.
struct Blk3 {
    const int8_t* N;       // [rows][k_pad]
    const int32_t* s;      // [rows]
    const double* w;       // [rows][2]
    int64_t rows;
    int64_t row0;          // global index of local row 0
};

// Kernel arguments of the fused 3-way pivot GEMM (KB-3W).  A unit computes the triples
// {p, m, n} with p in [p_lo,p_hi) of block bp (the pivot), m in [m_lo,m_hi) of bm (GEMM
// rows), n in [n_lo,n_hi) of bn (GEMM columns); same_pm => m > p, same_mn => n > m.
// `order` names the role (0 = p, 1 = m, 2 = n) in each canonical (sorted) slot.
struct Tally3Args {
    Blk3 bp, bm, bn;
    int64_t p_lo, p_hi, m_lo, m_hi, n_lo, n_hi;
    int32_t same_pm, same_mn, order, layout;   // layout: 0 in-block lexicographic,
                                               // 1 pair(p,m)-major x n, 2 dense box
    int32_t exact23;           // gamma == 2/3: CCC = double(T*U_p*U_m) * (U_n/D), D = 216 n_f^4
    int32_t exact52;           // exact23 and 72 n_f^3 < 2^52: T*U_p*U_m fits a double's mantissa
    double inv_d;              // 1 / (216 n_f^4)
    const int32_t* G;          // global pairwise G: G[min * ldG + max] (i < j valid)
    int64_t ldG;
    int64_t rec_base;          // subtracted from every record index (stages)
    int64_t k_pad;
    int32_t n_f, k_blocks, out_flags;
    int32_t permb;             // B rows arrive permuted within 8 (tmB is the 4-D view of
                               // make_tmap_b3): TMEM chunk columns (2j, 2j+1) hold n = j, j + 4
    uint32_t* tallies;         // [records][8]
    void* ccc;                 // [records][8] double or float
    unsigned long long* checksum;
    Compact cmp;               // used when compact != 0
    int32_t compact;
    int32_t ppair;             // single-block triangle: pivot pairs (PivotSched) -- the two CTAs
                               // of a pair share 128 rows m and take consecutive pivots
    unsigned long long* trace; // optional per-unit %globaltimer trace (diagnostics)
    // paper route (f4 ii): mode 1 stores this pass's form at forms[form_self * form_stride + rec]
    uint32_t* forms;
    int64_t form_stride;
    int32_t form_self, mode;
    // f4(ii) paper route (mode 3): masked marginals Mx[xi][p * ldG + x] = sum_{q: v_pq in xi} n_xq
    // and class counts cnt[xi][p] (xi = 0, 1, 2 for the paper's classes 1, 2, 3)
    const int32_t* mx[3];
    const int32_t* mcnt;
};

}  // namespace ccc
