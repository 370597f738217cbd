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

namespace ccc {

constexpr int kStages2 = 4;
constexpr int kABytes = kBM * kBK;  // 16 KB
constexpr int kBBytes = kBN * kBK;  // 32 KB
constexpr int kThreads2 = 192;
constexpr int kSmemBarOff2 = kStages2 * (kABytes + kBBytes);
constexpr int kSmem2 = kSmemBarOff2 + 256 + 1024;  // + barriers + alignment slack

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

__global__ void __launch_bounds__(kThreads2, 1)
tally2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const Tally2Args args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* smA = smem;
    uint8_t* smB = smem + kStages2 * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSmemBarOff2);
    uint64_t* empty = full + kStages2;
    uint64_t* tfull = empty + kStages2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    TriSched sch;
    sch.init(args.a_lo, args.nA, args.nB, args.diag);

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------------------ TMA producer
            uint32_t stage = 0, phase = 0;
            for (int64_t t = blockIdx.x;; t += gridDim.x) {
                int32_t bm, bn;
                if (!sch.get(t, bm, bn)) break;
                const int32_t arow = (int32_t)(args.a_lo + (int64_t)bm * kBM);
                const int32_t brow = bn * kBN;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], kABytes + kBBytes);
                    tma_load_2d(smA + stage * kABytes, &tmA, &full[stage], kb * kBK, arow);
                    tma_load_2d(smB + stage * kBBytes, &tmB, &full[stage], kb * kBK, brow);
                    if (++stage == kStages2) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = idesc_i8(kBM, kBN);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            const uint32_t a0 = smem_u32(smA), b0 = smem_u32(smB);
            for (int64_t t = blockIdx.x;; t += gridDim.x) {
                int32_t bm, bn;
                if (!sch.get(t, bm, bn)) break;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * kBN;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = a0 + stage * kABytes, sb = b0 + stage * kBBytes;
#pragma unroll
                    for (int k = 0; k < kBK / kUMMA_K; ++k)
                        mma_i8(d, smem_desc_sw128(sa + k * kUMMA_K),
                               smem_desc_sw128(sb + k * kUMMA_K), idesc, (kb | k) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == kStages2) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------------------- epilogue
        const uint32_t quad = warp & 3;            // TMEM lane quadrant of this warp
        const uint32_t row_in_tile = quad * 32 + lane;
        const int64_t nB = args.nB, a_end = args.a_lo + args.nA;
        const uint32_t fl = (uint32_t)args.out_flags;
        const bool want_t = fl & 1u, want_c64 = fl & 2u, want_c32 = fl & 4u, want_ck = fl & 8u;
        const uint32_t four_nf = 4u * (uint32_t)args.n_f;
        const double inv4nf = 1.0 / (4.0 * (double)args.n_f);
        unsigned long long ck_lo = 0, ck_hi = 0;
        uint32_t acc = 0, acc_phase = 0;
        for (int64_t t = blockIdx.x;; t += gridDim.x) {
            int32_t bm, bn;
            if (!sch.get(t, bm, bn)) break;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int64_t i = args.a_lo + (int64_t)bm * kBM + row_in_tile;
            const bool row_ok = i < a_end;
            int32_t s_i = 0;
            double wi0 = 0.0, wi1 = 0.0;
            if (row_ok) {
                s_i = __ldg(args.s_a + i);
                wi0 = __ldg(args.w_a + 2 * i);
                wi1 = __ldg(args.w_a + 2 * i + 1);
            }
            const int64_t rec_i = args.diag
                                      ? (i * (2 * nB - i - 1)) / 2 - i - 1 - args.rec_row_base
                                      : (i - args.a_lo) * nB;
            const uint32_t two_si = 2u * (uint32_t)s_i;
            const uint64_t gi = (uint64_t)(args.a_row0 + i);
            const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * kBN;
            for (int c = 0; c < kBN / 16; ++c) {
                uint32_t v[16];
                tmem_ld16(taddr + c * 16, v);
                tmem_ld_wait();
                const int64_t j0 = (int64_t)bn * kBN + c * 16;
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int64_t j = j0 + u;
                    const bool ok = row_ok && j < nB && (!args.diag || j > i);
                    if (!ok) continue;
                    const uint32_t g = v[u];
                    const int32_t s_j = __ldg(args.s_b + j);
                    const uint32_t two_sj = 2u * (uint32_t)s_j;
                    const uint32_t t11 = g, t10 = two_si - g, t01 = two_sj - g;
                    const uint32_t t00 = four_nf - two_si - two_sj + g;
                    const int64_t rec = rec_i + j;
                    if (want_t) st_v4_u32(args.tallies + 4 * rec, t00, t01, t10, t11);
                    if (want_c64 | want_c32) {
                        const double wj0 = __ldg(args.w_b + 2 * j);
                        const double wj1 = __ldg(args.w_b + 2 * j + 1);
                        const double c00 = (double)t00 * inv4nf * wi0 * wj0;
                        const double c01 = (double)t01 * inv4nf * wi0 * wj1;
                        const double c10 = (double)t10 * inv4nf * wi1 * wj0;
                        const double c11 = (double)t11 * inv4nf * wi1 * wj1;
                        if (want_c64) {
                            double* p = reinterpret_cast<double*>(args.ccc) + 4 * rec;
                            st_v2_f64(p, c00, c01);
                            st_v2_f64(p + 2, c10, c11);
                        } else {
                            float* p = reinterpret_cast<float*>(args.ccc) + 4 * rec;
                            st_v4_f32(p, (float)c00, (float)c01, (float)c10, (float)c11);
                        }
                    }
                    if (args.g_out) args.g_out[i * args.ldg + j] = (int32_t)g;
                    if (want_ck) {
                        const uint64_t gj = (uint64_t)(args.b_row0 + j);
                        ck_fold(ck_lo, ck_hi, (2ull << 60) | (gi << 40) | (gj << 20),
                                (uint64_t)t00 | ((uint64_t)t01 << 32),
                                (uint64_t)t10 | ((uint64_t)t11 << 32));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (want_ck) ck_flush(ck_lo, ck_hi, args.checksum);
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<512>(tmem_base);
}

// ------------------------------------------------------------------------- host side
cudaError_t launch_tally2(const CUtensorMap& tmA, const CUtensorMap& tmB, const Tally2Args& a,
                          int num_sms, cudaStream_t stream, int64_t* n_tiles_out) {
    TriSched sch;
    sch.init(a.a_lo, a.nA, a.nB, a.diag);
    const int64_t tiles = sch.total();
    if (n_tiles_out) *n_tiles_out = tiles;
    if (tiles == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(tally2_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
    if (e != cudaSuccess) return e;
    const int grid = (int)(tiles < num_sms ? tiles : num_sms);
    tally2_kernel<<<grid, kThreads2, kSmem2, stream>>>(tmA, tmB, a);
    return cudaGetLastError();
}

}  // namespace ccc
