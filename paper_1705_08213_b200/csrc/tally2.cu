// tally2.cu -- KB-2W: persistent tcgen05 kind::i8 tally GEMM with the fused 2-way
// CCC epilogue.
//
// Method (§2.1, Eq.2-3): with n_{iq} = rho_{i,q}(1) in {0,1,2} and
// rho_{i,q}(0) = 2 - n_{iq} (each entry holds exactly two alleles), the
// four pair tallies follow from ONE integer product G = N N^T:
//     T(1,1) = G_ij, T(1,0) = 2 s_i - G_ij, T(0,1) = 2 s_j - G_ij,
//     T(0,0) = 4 n_f - 2 s_i - 2 s_j + G_ij,            s_i = sum_q n_{iq}.
// This replaces the paper's popcount-in-ZGEMM "mGEMM2" with one int8 MAC
// per elementwise comparison on the 5th-generation tensor cores.
//
// Kernel structure (one CTA per SM, persistent over upper-triangular tiles):
//   warp 0 (1 thread) : TMA producer, 4-stage smem ring of A[128x128B] + B[256x128B]
//   warp 1            : TMEM allocator; 1 thread issues tcgen05.mma (M128 N256 K32)
//   warps 2..5        : epilogue, TMEM -> registers (tcgen05.ld 32x32b) -> tallies,
//                       fp64 CCC, stores of unique (i<j) records, checksum fold.
//   TMEM: 2 x 256 int32 accumulator columns (double-buffered: the MMA of tile t+1
//   runs while the epilogue drains tile t).
#include "sm100.cuh"
#include "common.cuh"
#include "internal.h"

#include <cstdio>
#include <cstdlib>

#ifndef CCC_PAIR_STAGES
#define CCC_PAIR_STAGES 6
#endif

namespace ccc {

__device__ __forceinline__ void ck_fold(unsigned long long& lo, unsigned long long& hi,
                                        uint64_t l0, uint64_t l1, uint64_t l2) {
    uint64_t h = kCkSeed;
    h = fmix64(h ^ l0);
    h = fmix64(h ^ l1);
    h = fmix64(h ^ l2);
    uint64_t dlo = h, dhi = fmix64(h ^ kCkHi);
    unsigned long long nlo = lo + dlo;
    hi += dhi + (nlo < lo ? 1ull : 0ull);
    lo = nlo;
}

__device__ __forceinline__ void ck_flush(unsigned long long lo, unsigned long long hi,
                                         unsigned long long* ck) {
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
        unsigned long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        unsigned long long nlo = lo + olo;
        hi += ohi + (nlo < lo ? 1ull : 0ull);
        lo = nlo;
    }
    if (lane_id() == 0 && (lo | hi)) {
        unsigned long long old = atomicAdd(&ck[0], lo);
        unsigned long long carry = (old + lo < old) ? 1ull : 0ull;
        atomicAdd(&ck[1], hi + carry);
    }
}

#ifndef CCC_EPI_WARPS
#define CCC_EPI_WARPS 4
#endif
constexpr int kEpiWarps2 = CCC_EPI_WARPS;          // 4 or 8 (1 or 2 per TMEM lane quadrant)
constexpr int kThreads2 = 64 + 32 * kEpiWarps2;    // producer, MMA, epilogue warps

template <int kPair>
struct Cfg2 {
    static constexpr int kTileM = 128 * kPair;     // tile rows (UMMA M = 128 / 256)
    static constexpr int kBRows = kBN / kPair;     // B rows held by each CTA
    static constexpr int kABytes = 128 * kBK;      // 16 KB of A per stage per CTA
    static constexpr int kBBytes = kBRows * kBK;   // B bytes per stage per CTA
    static constexpr int kStages = kPair == 2 ? CCC_PAIR_STAGES : 4;
    static constexpr int kBarOff = kStages * (kABytes + kBBytes);
    static constexpr int kSmem = kBarOff + 256 + 1024;
};

// f2 compaction: append one kept record (2-way key = i * 2^20 + j, global indices).
__device__ __forceinline__ void emit2(const Tally2Args& a, uint64_t key, uint32_t t00, uint32_t t01,
                                      uint32_t t10, uint32_t t11, double c00, double c01,
                                      double c10, double c11) {
    const unsigned long long slot = compact_slot(a.cmp.count);
    if (slot >= (unsigned long long)a.cmp.cap) return;
    a.cmp.keys[slot] = key;
    const uint32_t fl = (uint32_t)a.out_flags;
    if (fl & 1u) stg_128_u32(a.tallies + 4 * slot, t00, t01, t10, t11);
    if (fl & 2u) stg_256_f64(reinterpret_cast<double*>(a.ccc) + 4 * slot, c00, c01, c10, c11);
    else if (fl & 4u)
        stg_128_u32(reinterpret_cast<float*>(a.ccc) + 4 * slot, __float_as_uint((float)c00),
                    __float_as_uint((float)c01), __float_as_uint((float)c10), __float_as_uint((float)c11));
}

// kFull: the FULL headline output (tallies + fp64 CCC, gamma = 2/3 with 12 n_f^2 < 2^52, no
// raw G, no export, no checksum) as a flag-free epilogue: straight-line record code.
template <int kPair, bool kCompact, bool kSparse, bool kFull = false>
__global__ void __launch_bounds__(kThreads2, 1)
tally2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const Tally2Args args) {
    using C = Cfg2<kPair>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* smA = smem;
    uint8_t* smB = smem + C::kStages * C::kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rank = kPair == 2 ? cluster_ctarank() : 0u;  // 0 = leader CTA
    // tiles [t_lo, t_hi) of the schedule (t_hi = 0: all); f3 field-split waves use a range
    const int64_t unit0 = args.t_lo + blockIdx.x / kPair, units = gridDim.x / kPair;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], kPair);   // leader: expect_tx arrive (+ follower arrive)
            mbar_init(&empty[s], 1);      // one (multicast) MMA commit per use
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpiWarps2 * kPair);  // one arrive per epilogue warp of the pair
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (kPair == 2) tmem_alloc_pair<512>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    if constexpr (kPair == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    TriSched sch;
    sch.init(args.a_lo, args.nA, args.nB, args.diag, C::kTileM, args.sup_rows, args.sup_cols);

    if (warp == 0) {
        {
            // ------------------------------------------------------------ TMA producer
            // whole warp walks the loop (uniform coordinates); one elected lane issues
            uint32_t stage = 0, phase = 0;
            const uint64_t pol = policy_evict_last();
            for (int64_t t = unit0;; t += units) {
                int32_t bm, bn;
                if ((args.t_hi > 0 && t >= args.t_hi) || !sch.get(t, bm, bn)) break;
                const int32_t arow = (int32_t)(args.a_lo + (int64_t)bm * C::kTileM + rank * 128);
                const int32_t brow = (int32_t)sch.b_lo + bn * kBN + (int32_t)rank * C::kBRows;
                if (args.trace && rank == 0 && lane == 0) args.trace[8 * t + 6] = globaltimer();

                // odd waves walk K backwards: they start on the k-blocks the previous wave
                // touched last, which are still in L2 (the MMA accumulates in any order)
                const bool rev = args.k_alternate && (((t - unit0) / units) & 1);
                for (int32_t kk = 0; kk < args.k_blocks; ++kk) {
                    const int32_t kb = rev ? args.k_blocks - 1 - kk : kk;
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smA + stage * C::kABytes;
                    uint8_t* sb = smB + stage * C::kBBytes;
                    if (elect_one()) {
#ifdef CCC_D2_NOTMA   // diagnostics: no operand loads (stale tiles; timing only)
                        if constexpr (kPair == 2) {
                            if (rank == 0) mbar_arrive(&full[stage]);
                            else mbar_arrive_cluster(mapa_shared(smem_u32(&full[stage]), 0));
                        } else {
                            mbar_arrive(&full[stage]);
                        }
                        if (true) {} else
#endif
                        if constexpr (kPair == 2) {
                            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
                            if (rank == 0)
                                mbar_arrive_expect_tx(&full[stage], 2 * (C::kABytes + C::kBBytes));
                            else
                                mbar_arrive_cluster(fb);
                            tma_load_2d_pair(sa, &tmA, fb, kb * kBK, arow, pol);
                            tma_load_2d_pair(sb, &tmB, fb, kb * kBK, brow, pol);
                        } else {
                            mbar_arrive_expect_tx(&full[stage], C::kABytes + C::kBBytes);
                            tma_load_2d(sa, &tmA, &full[stage], kb * kBK, arow, pol);
                            tma_load_2d(sb, &tmB, &full[stage], kb * kBK, brow, pol);
                        }
                    }
                    __syncwarp();
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ------------------------------------------------------------ MMA issuer
            // The whole warp walks the loop (descriptors stay warp-uniform, in uniform
            // registers); one elected lane issues each tcgen05.mma / commit.
            constexpr uint32_t idesc = idesc_i8(C::kTileM, kBN);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            const uint64_t a_desc0 = smem_desc_sw128(smem_u32(smA));
            const uint64_t b_desc0 = smem_desc_sw128(smem_u32(smB));
            for (int64_t t = unit0;; t += units) {
                int32_t bm, bn;
                if ((args.t_hi > 0 && t >= args.t_hi) || !sch.get(t, bm, bn)) break;
                unsigned long long* tr = (args.trace && lane == 0) ? args.trace + 8 * t : nullptr;
                if (tr) tr[0] = globaltimer();
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                if (tr) tr[1] = globaltimer();
                const uint32_t d = tmem_base + acc * kBN;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    // descriptor start address is in 16-B units in the low bits: advancing
                    // the operand by x bytes adds x >> 4 (no carry out of the 14-bit field
                    // inside the CTA's shared window)
                    const uint64_t ad = a_desc0 + ((stage * C::kABytes) >> 4);
                    const uint64_t bd = b_desc0 + ((stage * C::kBBytes) >> 4);
                    if (elect_one()) {
#ifdef CCC_D2_NOMMA   // diagnostics: no MMAs (the accumulator holds stale values; timing only)
                        if (false)
#endif
#pragma unroll
                        for (int k = 0; k < kBK / kUMMA_K; ++k) {
                            if constexpr (kPair == 2)
                                mma_i8_pair(d, ad + (k * kUMMA_K >> 4), bd + (k * kUMMA_K >> 4), idesc, (kb | k) != 0);
                            else mma_i8(d, ad + (k * kUMMA_K >> 4), bd + (k * kUMMA_K >> 4), idesc, (kb | k) != 0);
                        }
                        if constexpr (kPair == 2) mma_commit_pair(&empty[stage], 3);
                        else mma_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == C::kStages) { stage = 0; phase ^= 1; }
                }
                if (elect_one()) {
                    if constexpr (kPair == 2) mma_commit_pair(&tfull[acc], 3);
                    else mma_commit(&tfull[acc]);
                }
                __syncwarp();
                if (tr) tr[2] = globaltimer();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
        __syncwarp();
    } else if constexpr (kSparse) {
        // ------------------------------------------------------ sparse epilogue (f1)
        // X is group-interleaved (16 rows n, then 16 rows v per group of 16 vectors), so
        // each epilogue warp's TMEM quadrant is one group of vectors i: lanes 0-15 hold
        // rows n_i, lanes 16-31 rows v_i.  Per 32-column group (vectors j: columns 0-15
        // n_j, 16-31 v_j) lane t < 16 holds G = n_i.n_j, H = n_i.v_j and lane t + 16
        // H' = v_i.n_j, C = v_i.v_j = c_ij; one shuffle round hands thread t < 16 all four
        // for j = 0..7 and thread t + 16 for j = 8..15.  With rho(1) = n, rho(0) = 2v - n:
        //   T11 = G, T10 = 2H - G, T01 = 2H' - G, T00 = 4C - 2H - 2H' + G
        //   CCC(a,b) = T(a,b) / (4 c_ij) * w_i(a) * w_j(b)   (reading A-17; 0 if c_ij = 0)
        const uint32_t quad = warp & 3;
        const bool low = lane < 16;
        const uint32_t fl = (uint32_t)args.out_flags;
        const bool want_t = fl & 1u, want_c64 = fl & 2u, want_c32 = fl & 4u, want_ck = fl & 8u;
        const bool want_c = want_c64 | want_c32;
        const int64_t nBv = args.nBv;
        const uint32_t tempty_leader = kPair == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        unsigned long long ck_lo = 0, ck_hi = 0;
        uint32_t acc = 0, acc_phase = 0;
        for (int64_t t = unit0;; t += units) {
            int32_t bm, bn;
            if ((args.t_hi > 0 && t >= args.t_hi) || !sch.get(t, bm, bn)) break;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t xrow = args.a_lo + (int64_t)bm * C::kTileM + rank * 128 + quad * 32;
            const int64_t i_w = xrow >> 1;                    // first vector of my group
            const int64_t i = i_w + (lane & 15);
            const bool row_ok = i >= args.v_lo && i < args.v_hi;
            const int64_t ic = row_ok ? i : args.v_lo;
            const double wi0 = __ldg(args.w_a + 2 * ic), wi1 = __ldg(args.w_a + 2 * ic + 1);
            const int64_t rec_i = args.diag ? (i * (2 * nBv - i - 1)) / 2 - i - 1 - args.rec_row_base
                                            : (i - args.v_lo) * nBv;
            const uint64_t gi = (uint64_t)(args.a_row0 + i);
            const bool any_row = __any_sync(0xffffffffu, row_ok);
            const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * kBN;
            for (int cg = 0; cg < kBN / 32; ++cg) {
                const int64_t j0 = ((int64_t)bn * kBN + cg * 32) >> 1;   // first vector j
                if (!any_row || j0 >= nBv || (args.diag && j0 + 15 <= i_w)) continue;  // uniform
                uint32_t v[32];
                tmem_ld16(taddr + cg * 32, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(taddr + cg * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld_wait();
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t r0 = __shfl_xor_sync(0xffffffffu, low ? v[8 + k] : v[k], 16);
                    const uint32_t r1 = __shfl_xor_sync(0xffffffffu, low ? v[24 + k] : v[16 + k], 16);
                    const uint32_t G = low ? v[k] : r0, H = low ? v[16 + k] : r1;
                    const uint32_t Hp = low ? r0 : v[8 + k], Cc = low ? r1 : v[24 + k];
                    const int64_t j = j0 + (low ? k : 8 + k);
                    if (!(row_ok && j < nBv && (!args.diag || j > i))) continue;
                    const uint32_t t11 = G, t10 = 2u * H - G, t01 = 2u * Hp - G;
                    const uint32_t t00 = 4u * Cc - 2u * H - 2u * Hp + G;
                    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
                    if ((want_c || kCompact) && Cc != 0u) {
                        const double inv = 1.0 / (4.0 * (double)Cc);
                        const double wj0 = __ldg(args.w_b + 2 * j), wj1 = __ldg(args.w_b + 2 * j + 1);
                        const double a0 = wi0 * inv, a1 = wi1 * inv;
                        c00 = (double)t00 * a0 * wj0;
                        c01 = (double)t01 * a0 * wj1;
                        c10 = (double)t10 * a1 * wj0;
                        c11 = (double)t11 * a1 * wj1;
                    }
                    const uint64_t gj = (uint64_t)(args.b_row0 + j);
                    if constexpr (kCompact) {
                        if (fmax(fmax(c00, c01), fmax(c10, c11)) > args.cmp.thr)
                            emit2(args, (gi << 20) | gj, t00, t01, t10, t11, c00, c01, c10, c11);
                    } else {
                        const int64_t rec = rec_i + j;
                        if (want_t) stg_128_u32(args.tallies + 4 * rec, t00, t01, t10, t11);
                        if (want_c64)
                            stg_256_f64(reinterpret_cast<double*>(args.ccc) + 4 * rec, c00, c01, c10, c11);
                        else if (want_c32)
                            stg_128_u32(reinterpret_cast<float*>(args.ccc) + 4 * rec,
                                        __float_as_uint((float)c00), __float_as_uint((float)c01),
                                        __float_as_uint((float)c10), __float_as_uint((float)c11));
                    }
                    if (want_ck)
                        ck_fold(ck_lo, ck_hi, (2ull << 60) | (gi << 40) | (gj << 20),
                                (uint64_t)t00 | ((uint64_t)t01 << 32), (uint64_t)t10 | ((uint64_t)t11 << 32));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kPair == 2 && rank != 0) mbar_arrive_cluster(tempty_leader + acc * 8u);
                else mbar_arrive(&tempty[acc]);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (want_ck) ck_flush(ck_lo, ck_hi, args.checksum);
    } else {
        // ---------------------------------------------------------------- epilogue
        // Each warp drains its 32-lane TMEM quadrant with tcgen05.ld.16x256b: per 8-column
        // chunk a thread holds 2 consecutive records of 4 rows, so tallies (16 B/record)
        // and fp64 CCC (32 B/record) leave as 256-bit stores of whole L2 sectors straight
        // from registers -- no shared-memory staging, which would compete with the TMA
        // fills and tensor-core operand reads of the mainloop.
        const uint32_t quad = warp & 3;            // TMEM lane quadrant of this warp
        const int c_begin = ((warp - 2) / 4) * (kBN / 8 / (kEpiWarps2 / 4));  // my column chunks
        const int c_end = c_begin + kBN / 8 / (kEpiWarps2 / 4);
        const int64_t nB = args.nB, a_end = args.a_lo + args.nA;
        const uint32_t fl = (uint32_t)args.out_flags;
        const bool want_t = kFull || (fl & 1u), want_c64 = kFull || (fl & 2u);
        const bool want_c32 = !kFull && (fl & 4u), want_ck = !kFull && (fl & 8u);
        const bool want_c = want_c64 | want_c32;
        const uint32_t nf = (uint32_t)args.n_f;
        const uint32_t four_nf = 4u * nf;
        const double inv4nf = 1.0 / (4.0 * (double)args.n_f);
        const bool exact23 = kFull || args.exact23 != 0;
        // gamma = 2/3 and 12 n_f^2 < 2^52: the single-DFMA cell form below
        const bool exact52 = kFull || (exact23 && (uint64_t)12 * nf * nf < (1ull << 52));
        const uint32_t tempty_leader = kPair == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        const int32_t cpair = 2 * (int32_t)(lane & 3);   // my 2 columns within a chunk
        unsigned long long ck_lo = 0, ck_hi = 0;
        uint32_t acc = 0, acc_phase = 0;
        for (int64_t t = unit0;; t += units) {
            int32_t bm, bn;
            if ((args.t_hi > 0 && t >= args.t_hi) || !sch.get(t, bm, bn)) break;
            unsigned long long* tr = (args.trace && warp == 2 && rank == 0) ? args.trace + 8 * t : nullptr;
            if (tr && lane == 0) tr[3] = globaltimer();
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (tr && lane == 0) tr[4] = globaltimer();
            // my 4 rows: r = quad*32 + h*16 + e*8 + lane/4, h, e in {0,1}
            int64_t rec_r[4];
            int32_t jlo_r[4], jhi_r[4];
            uint32_t two_si[4], ui0[4], ui1[4];
            double wi0[4], wi1[4];
            uint64_t gi[4];
            bool my_any = false;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t i = args.a_lo + (int64_t)bm * C::kTileM + rank * 128 + quad * 32 +
                                  (r >> 1) * 16 + (r & 1) * 8 + (lane >> 2);
                const bool row_ok = i < a_end;
                two_si[r] = row_ok ? 2u * (uint32_t)__ldg(args.s_a + i) : 0u;
                ui0[r] = nf + (two_si[r] >> 1);          // U_i(0) = 3 n_f - S_i(0) = n_f + s_i
                ui1[r] = 3u * nf - (two_si[r] >> 1);     // U_i(1) = 3 n_f - s_i
                wi0[r] = (row_ok && !exact23) ? __ldg(args.w_a + 2 * i) * inv4nf : 0.0;   // w_i(0)/(4n_f)
                wi1[r] = (row_ok && !exact23) ? __ldg(args.w_a + 2 * i + 1) * inv4nf : 0.0;
                rec_r[r] = args.diag ? (i * (2 * nB - i - 1)) / 2 - i - 1 - args.rec_row_base
                                     : (i - args.a_lo) * nB;
#ifdef CCC_D2_ALIGNADDR   // diagnostics: every row's records start at a multiple of 8 (timing only)
                rec_r[r] = (rec_r[r] + 8) & ~(int64_t)7;
#endif
#ifdef CCC_D2_ALIGN2ADDR  // diagnostics: every row's records start at a multiple of 2 (timing only)
                rec_r[r] = (rec_r[r] + 2) & ~(int64_t)1;
#endif
                jlo_r[r] = args.diag ? (int32_t)(i + 1) : 0;
                jhi_r[r] = row_ok ? (int32_t)nB : 0;
                gi[r] = (uint64_t)(args.a_row0 + i);
                my_any |= row_ok && jlo_r[r] < jhi_r[r];
            }
            const bool any_row = __any_sync(0xffffffffu, my_any);
            const int32_t warp_jlo = __shfl_sync(0xffffffffu, jlo_r[0], 0);
            const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * kBN;
            for (int c = c_begin; c < c_end; ++c) {
                const int32_t j0 = bn * kBN + c * 8;
                if (!any_row || j0 >= nB || j0 + 8 <= warp_jlo) continue;  // warp-uniform
                uint32_t va[4], vb[4];
#ifdef CCC_D2_NOTMEMLD
                for (int x = 0; x < 4; ++x) { va[x] = lane + x + c; vb[x] = lane * 3 + x; }   // diagnostics
#else
                tmem_ld_16x256(taddr + c * 8, va);                  // lanes +0..15
                tmem_ld_16x256(taddr + (16u << 16) + c * 8, vb);    // lanes +16..31
#endif
                const int32_t jA = j0 + cpair, jB = jA + 1;
                const int32_t jAc = jA < nB ? jA : (int32_t)nB - 1;
                const int32_t jBc = jB < nB ? jB : (int32_t)nB - 1;
                const uint32_t two_sA = 2u * (uint32_t)__ldg(args.s_b + jAc);
                const uint32_t two_sB = 2u * (uint32_t)__ldg(args.s_b + jBc);
                // column factors: general gamma -> w_j(b); gamma = 2/3 -> U_j(b) / (36 n_f^3)
                // with the integer U_j(0) = n_f + s_j, U_j(1) = 3 n_f - s_j
                double wA0 = 0.0, wA1 = 0.0, wB0 = 0.0, wB1 = 0.0;
                double mA0 = 0.0, mA1 = 0.0, mB0 = 0.0, mB1 = 0.0;
                if (want_c || kCompact) {
#ifdef CCC_D2_NOFP64
                    if (false) {
#else
                    if (exact23) {
#endif
                        const uint32_t sAj = two_sA >> 1, sBj = two_sB >> 1;
                        wA0 = u32_to_f64(nf + sAj) * args.inv_d;
                        wA1 = u32_to_f64(3u * nf - sAj) * args.inv_d;
                        wB0 = u32_to_f64(nf + sBj) * args.inv_d;
                        wB1 = u32_to_f64(3u * nf - sBj) * args.inv_d;
                        mA0 = -4503599627370496.0 * wA0;
                        mA1 = -4503599627370496.0 * wA1;
                        mB0 = -4503599627370496.0 * wB0;
                        mB1 = -4503599627370496.0 * wB1;
                    } else {
                        wA0 = __ldg(args.w_b + 2 * jAc);
                        wA1 = __ldg(args.w_b + 2 * jAc + 1);
                        wB0 = __ldg(args.w_b + 2 * jBc);
                        wB1 = __ldg(args.w_b + 2 * jBc + 1);
                    }
                }
                tmem_ld_wait();
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint32_t gA = (r >> 1) ? vb[(r & 1) * 2] : va[(r & 1) * 2];
                    const uint32_t gB = (r >> 1) ? vb[(r & 1) * 2 + 1] : va[(r & 1) * 2 + 1];
                    const bool okA = jA >= jlo_r[r] && jA < jhi_r[r];
                    const bool okB = jB >= jlo_r[r] && jB < jhi_r[r];
                    if (!kFull && args.xp_ptrs && (okA | okB)) {
                        // f3 field split: this field slice's partial G of the tile goes
                        // straight to the owner's slot (a peer-mapped pointer over NVLink
                        // on a multi-GPU run), overlapped with the MMAs of later tiles
                        const int64_t world = args.xp_world;
                        const int64_t slot = (t - args.t_lo) / world;
                        int32_t* dst = args.xp_ptrs[t % world] + ((slot * world + args.xp_rank) << 16);
                        const int32_t trow = (int32_t)(rank * 128 + quad * 32 + (r >> 1) * 16 + (r & 1) * 8 +
                                                       (lane >> 2));
                        const int32_t tcol = c * 8 + cpair;
                        *reinterpret_cast<int2*>(dst + trow * kBN + tcol) = make_int2((int32_t)gA, (int32_t)gB);
                        continue;
                    }
                    if (!(okA | okB)) continue;
                    // Eq.2 tallies from G (rho(0) = 2 - rho(1))
                    const uint32_t a11 = gA, a10 = two_si[r] - gA, a01 = two_sA - gA;
                    const uint32_t a00 = four_nf - two_si[r] - two_sA + gA;
                    const uint32_t b11 = gB, b10 = two_si[r] - gB, b01 = two_sB - gB;
                    const uint32_t b00 = four_nf - two_si[r] - two_sB + gB;
                    const int64_t recA = rec_r[r] + jA;
                    // Eq.3: CCC(a,b) = T(a,b) / (4 n_f) * w_i(a) * w_j(b).  For gamma = 2/3,
                    // w(a) = U(a) / (3 n_f) with integer U, so CCC = T U_i(a) U_j(b) / (36 n_f^3):
                    // T * U_i(a) < 2^53 is exact in a double and one DMUL per cell remains
                    // (FP64 issue rate is the scarce resource of this epilogue on B200).
                    double ca00 = 0, ca01 = 0, ca10 = 0, ca11 = 0, cb00 = 0, cb01 = 0, cb10 = 0, cb11 = 0;
                    if (want_c || kCompact) {
#ifdef CCC_D2_NOFP64
                        if (true) {   // diagnostics: integer-only stand-in for the CCC cells
                            const uint32_t u0 = ui0[r], u1 = ui1[r];
                            ca00 = magic52((uint64_t)a00 * u0); ca01 = magic52((uint64_t)a01 * u0);
                            ca10 = magic52((uint64_t)a10 * u1); ca11 = magic52((uint64_t)a11 * u1);
                            cb00 = magic52((uint64_t)b00 * u0); cb01 = magic52((uint64_t)b01 * u0);
                            cb10 = magic52((uint64_t)b10 * u1); cb11 = magic52((uint64_t)b11 * u1);
                        } else
#endif
                        if (exact52) {
                            // P = T U_i(a) < 12 n_f^2 < 2^52: the double 2^52 + P is P's bits
                            // under exponent 0x433, so CCC = P w = fma(2^52 + P, w, -2^52 w):
                            // one rounding (as before), one FP64 op and no I2F (the XU pipe
                            // was the limiter of this epilogue)
                            const uint32_t u0 = ui0[r], u1 = ui1[r];
                            ca00 = __fma_rn(magic52((uint64_t)a00 * u0), wA0, mA0);
                            ca01 = __fma_rn(magic52((uint64_t)a01 * u0), wA1, mA1);
                            ca10 = __fma_rn(magic52((uint64_t)a10 * u1), wA0, mA0);
                            ca11 = __fma_rn(magic52((uint64_t)a11 * u1), wA1, mA1);
                            cb00 = __fma_rn(magic52((uint64_t)b00 * u0), wB0, mB0);
                            cb01 = __fma_rn(magic52((uint64_t)b01 * u0), wB1, mB1);
                            cb10 = __fma_rn(magic52((uint64_t)b10 * u1), wB0, mB0);
                            cb11 = __fma_rn(magic52((uint64_t)b11 * u1), wB1, mB1);
                        } else if (exact23) {
                            const uint64_t u0 = ui0[r], u1 = ui1[r];
                            ca00 = (double)(a00 * u0) * wA0;
                            ca01 = (double)(a01 * u0) * wA1;
                            ca10 = (double)(a10 * u1) * wA0;
                            ca11 = (double)(a11 * u1) * wA1;
                            cb00 = (double)(b00 * u0) * wB0;
                            cb01 = (double)(b01 * u0) * wB1;
                            cb10 = (double)(b10 * u1) * wB0;
                            cb11 = (double)(b11 * u1) * wB1;
                        } else {
                            ca00 = (double)a00 * wi0[r] * wA0;
                            ca01 = (double)a01 * wi0[r] * wA1;
                            ca10 = (double)a10 * wi1[r] * wA0;
                            ca11 = (double)a11 * wi1[r] * wA1;
                            cb00 = (double)b00 * wi0[r] * wB0;
                            cb01 = (double)b01 * wi0[r] * wB1;
                            cb10 = (double)b10 * wi1[r] * wB0;
                            cb11 = (double)b11 * wi1[r] * wB1;
                        }
                    }
                    if constexpr (kCompact) {
                        // f2: keep a record iff its largest CCC cell exceeds the threshold
                        const Compact& cm = args.cmp;
                        const double mA = fmax(fmax(ca00, ca01), fmax(ca10, ca11));
                        const double mB = fmax(fmax(cb00, cb01), fmax(cb10, cb11));
                        if (okA && mA > cm.thr)
                            emit2(args, (gi[r] << 20) | (uint64_t)(args.b_row0 + jA), a00, a01, a10, a11,
                                  ca00, ca01, ca10, ca11);
                        if (okB && mB > cm.thr)
                            emit2(args, (gi[r] << 20) | (uint64_t)(args.b_row0 + jB), b00, b01, b10, b11,
                                  cb00, cb01, cb10, cb11);
                    } else {
#ifdef CCC_D2_NOSTORE
                    const bool stA = okA && recA < 0, stB = okB && recA < 0;   // diagnostics
#else
                    const bool stA = okA, stB = okB;
#endif
                    if (want_t) {
                        uint32_t* p = args.tallies + 4 * recA;
                        if (stA && stB && !(recA & 1)) {
                            stg_256_u32(p, a00, a01, a10, a11, b00, b01, b10, b11);
                        } else {
                            if (stA) stg_128_u32(p, a00, a01, a10, a11);
                            if (stB) stg_128_u32(p + 4, b00, b01, b10, b11);
                        }
                    }
                    if (want_c) {
                        if (want_c64) {
                            double* p = reinterpret_cast<double*>(args.ccc) + 4 * recA;
#ifdef CCC_D2_CCC_NOALLOC   // experiment: the fp64 CCC half of the records bypasses L1 allocation
                            stg_256_f64_if(stA, p, ca00, ca01, ca10, ca11);
                            stg_256_f64_if(stB, p + 4, cb00, cb01, cb10, cb11);
#else
                            if constexpr (kFull) {   // branch-free
#if defined(CCC_D2_NOCCCST)   // diagnostics: CCC computed, never stored (kept alive by a test)
                                const bool never = recA < -1;
                                stg_256_f64_p(never && stA, p, ca00, ca01, ca10, ca11);
                                stg_256_f64_p(never && stB, p + 4, cb00, cb01, cb10, cb11);
#elif defined(CCC_D2_CCCCONST)   // diagnostics: CCC bytes stored, no FP64 / 64-bit math
                                stg_256_f64_p(stA, p, magic52(a00), magic52(a01), magic52(a10), magic52(a11));
                                stg_256_f64_p(stB, p + 4, magic52(b00), magic52(b01), magic52(b10), magic52(b11));
#else
                                stg_256_f64_p(stA, p, ca00, ca01, ca10, ca11);
                                stg_256_f64_p(stB, p + 4, cb00, cb01, cb10, cb11);
#endif
                            } else {
                                if (stA) stg_256_f64(p, ca00, ca01, ca10, ca11);
                                if (stB) stg_256_f64(p + 4, cb00, cb01, cb10, cb11);
                            }
#endif
                        } else {
                            float* p = reinterpret_cast<float*>(args.ccc) + 4 * recA;
                            if (stA && stB && !(recA & 1)) {
                                stg_256_u32(p, __float_as_uint((float)ca00), __float_as_uint((float)ca01),
                                            __float_as_uint((float)ca10), __float_as_uint((float)ca11),
                                            __float_as_uint((float)cb00), __float_as_uint((float)cb01),
                                            __float_as_uint((float)cb10), __float_as_uint((float)cb11));
                            } else {
                                if (stA)
                                    stg_128_u32(p, __float_as_uint((float)ca00), __float_as_uint((float)ca01),
                                                __float_as_uint((float)ca10), __float_as_uint((float)ca11));
                                if (stB)
                                    stg_128_u32(p + 4, __float_as_uint((float)cb00), __float_as_uint((float)cb01),
                                                __float_as_uint((float)cb10), __float_as_uint((float)cb11));
                            }
                        }
                    }
                    }
                    if (!kFull && args.g_out) {
                        const int64_t row = (int64_t)(gi[r] - (uint64_t)args.a_row0);
                        if (okA) args.g_out[row * args.ldg + jA] = (int32_t)gA;
                        if (okB) args.g_out[row * args.ldg + jB] = (int32_t)gB;
                    }
                    if (want_ck) {
                        if (okA)
                            ck_fold(ck_lo, ck_hi,
                                    (2ull << 60) | (gi[r] << 40) | ((uint64_t)(args.b_row0 + jA) << 20),
                                    (uint64_t)a00 | ((uint64_t)a01 << 32), (uint64_t)a10 | ((uint64_t)a11 << 32));
                        if (okB)
                            ck_fold(ck_lo, ck_hi,
                                    (2ull << 60) | (gi[r] << 40) | ((uint64_t)(args.b_row0 + jB) << 20),
                                    (uint64_t)b00 | ((uint64_t)b01 << 32), (uint64_t)b10 | ((uint64_t)b11 << 32));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (tr && lane == 0) tr[5] = globaltimer();
            if (lane == 0) {
                if (kPair == 2 && rank != 0) mbar_arrive_cluster(tempty_leader + acc * 8u);
                else mbar_arrive(&tempty[acc]);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (want_ck) ck_flush(ck_lo, ck_hi, args.checksum);
    }

    tc_fence_before();
    if constexpr (kPair == 2) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        if constexpr (kPair == 2) tmem_dealloc_pair<512>(tmem_base);
        else tmem_dealloc<512>(tmem_base);
    }
}

// ------------------------------------------------------------------------- host side
// Diagnostic knobs (1-CTA variant, super-tile shape, K direction, per-tile trace) exist
// only in builds with -DCCC_DIAG (scripts/); the product library ignores the environment,
// so the field-split export and finish kernels always share one tile schedule.
static int pair_mode() {
#ifdef CCC_DIAG
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("CCC_TALLY2_CTA");
        mode = (e && e[0] == '1') ? 1 : 2;
    }
    return mode;
#else
    return 2;
#endif
}

int tally2_tile_rows() { return pair_mode() == 2 ? 256 : 128; }
int tally2_b_box_rows() { return pair_mode() == 2 ? Cfg2<2>::kBRows : Cfg2<1>::kBRows; }

cudaError_t launch_tally2(const CUtensorMap& tmA, const CUtensorMap& tmB, const Tally2Args& a,
                          int num_sms, cudaStream_t stream, int64_t* n_tiles_out) {
    const int pm = pair_mode();
    TriSched sch;
    Tally2Args a2 = a;
#ifdef CCC_DIAG
    {
        const char* e = getenv("CCC_SUPER");   // "rows,cols" in elements
        if (e) sscanf(e, "%d,%d", &a2.sup_rows, &a2.sup_cols);
        const char* ka = getenv("CCC_KALT");
        if (ka) a2.k_alternate = atoi(ka);
        const char* tre = getenv("CCC_TRACE_PTR");   // diagnostics: device pointer (decimal)
        a2.trace = tre ? reinterpret_cast<unsigned long long*>(strtoull(tre, nullptr, 10)) : nullptr;
    }
#endif
    sch.init(a.a_lo, a.nA, a.nB, a.diag, (pm == 2 || a.sparse) ? Cfg2<2>::kTileM : Cfg2<1>::kTileM,
             a2.sup_rows, a2.sup_cols);
    const int64_t all_tiles = sch.total();
    const int64_t t_end = (a.t_hi > 0 && a.t_hi < all_tiles) ? a.t_hi : all_tiles;
    const int64_t tiles = t_end > a.t_lo ? t_end - a.t_lo : 0;   // f3 waves: a range
    if (n_tiles_out) *n_tiles_out = tiles;
    if (tiles == 0) return cudaSuccess;
    if (pm == 1 && !a.sparse) {
        auto kern = a.compact ? tally2_kernel<1, true, false> : tally2_kernel<1, false, false>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Cfg2<1>::kSmem);
        if (e != cudaSuccess) return e;
        const int grid = (int)(tiles < num_sms ? tiles : num_sms);
        kern<<<grid, kThreads2, Cfg2<1>::kSmem, stream>>>(tmA, tmB, a2);
        return cudaGetLastError();
    }
    const bool full = !a.sparse && !a.compact && a.out_flags == 3 && a.exact23 && !a.g_out && !a.xp_ptrs &&
                      (uint64_t)12 * (uint64_t)a.n_f * (uint64_t)a.n_f < (1ull << 52);
    auto kern = a.sparse ? (a.compact ? tally2_kernel<2, true, true> : tally2_kernel<2, false, true>)
                : full   ? tally2_kernel<2, false, false, true>
                         : (a.compact ? tally2_kernel<2, true, false> : tally2_kernel<2, false, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg2<2>::kSmem);
    if (e != cudaSuccess) return e;
    const int64_t pairs = num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * (tiles < pairs ? tiles : pairs)));
    cfg.blockDim = dim3(kThreads2);
    cfg.dynamicSmemBytes = Cfg2<2>::kSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, a2);
}

}  // namespace ccc
