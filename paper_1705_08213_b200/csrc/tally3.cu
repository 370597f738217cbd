// tally3.cu -- KB-3W: per-pivot Hadamard-weighted tcgen05 kind::i8 GEMM with the
// fused 3-way CCC epilogue (stages a8).
//
// Method (§2.2, Eq.4-5): for a pivot vector i (the FIRST index of the
// triple, so that a stage = a contiguous i-range = a contiguous slice of the
// lexicographic result array, cf. stages P:621-626),
//     G3_ijk = sum_q n_iq n_jq n_kq = ((N_J o n_i) N_K^T)_jk,
// one GEMM whose A operand is the Hadamard product of a row block of N with the
// pivot row.  All eight cells follow from G3, the pairwise G (precomputed by KB-2W)
// and s by inclusion-exclusion (rho(0) = 2 - rho(1)):
//     T111 = G3, T110 = 2G_ij - G3, T101 = 2G_ik - G3, T011 = 2G_jk - G3,
//     T100 = 4s_i - 2G_ij - 2G_ik + G3, T010 = 4s_j - 2G_ij - 2G_jk + G3,
//     T001 = 4s_k - 2G_ik - 2G_jk + G3,
//     T000 = 8n_f - 4(s_i+s_j+s_k) + 2(G_ij+G_ik+G_jk) - G3.
// The paper instead runs three masked mGEMM3 per pivot (Table 1); this
// needs one int8 MAC per unique 3-way comparison.
//
// Work unit = (row tile J of 128 j's, column tile K of 256 k's, pivot i); units are
// ordered tile-outer / pivot-inner so the ~148 concurrent CTAs share the same N_J,
// N_K panels in L2 and differ only in their 128-byte pivot rows.
// Warp roles: 0 TMA producer (A, B tiles + pivot chunk), 1 TMEM alloc + MMA issuer,
// 2..5 epilogue, 6..9 transform (A <- A o n_i in shared memory, in place).
#include "sm100.cuh"
#include "common.cuh"
#include "internal.h"

namespace ccc {

constexpr int kStages3 = 4;
constexpr int kABytes3 = kBM * kBK;  // 16 KB
constexpr int kBBytes3 = kBN * kBK;  // 32 KB
constexpr int kPivBytes = kBK;       // 128 B of the pivot row per stage
constexpr int kEpiWarps3 = 8;                                 // 2 per TMEM lane quadrant
constexpr int kXfWarps3 = 4;                                  // transform warps (1 row each lane)
constexpr int kThreads3 = 32 * (2 + kEpiWarps3 + kXfWarps3);  // 448
constexpr int kPivOff3 = kStages3 * (kABytes3 + kBBytes3);
constexpr int kBarOff3 = kPivOff3 + kStages3 * kPivBytes;
constexpr int kSmem3 = kBarOff3 + 256 + 1024;

struct PivotSched {
    TriSched tiles;
    int64_t n_v, i_begin, i_end, tt, base, cnt;
    int32_t J, K;

    __host__ __device__ int64_t pivots(int32_t Jt, int32_t Kt) const {
        int64_t jmax = (int64_t)Jt * kBM + kBM - 1;
        if (jmax > n_v - 1) jmax = n_v - 1;
        int64_t kmax = (int64_t)Kt * kBN + kBN - 1;
        if (kmax > n_v - 1) kmax = n_v - 1;
        int64_t imax = jmax < kmax - 1 ? jmax : kmax - 1;  // pivots i < imax
        int64_t hi = i_end < imax ? i_end : imax;
        return hi > i_begin ? hi - i_begin : 0;
    }
    __host__ __device__ void init(int64_t n_v_, int64_t ib, int64_t ie) {
        n_v = n_v_;
        i_begin = ib;
        i_end = ie;
        tiles.init(0, n_v, n_v, 1);
        tt = 0;
        base = 0;
        cnt = 0;
        J = K = 0;
        if (tiles.get(0, J, K)) cnt = pivots(J, K);
        else tt = -1;
    }
    __host__ __device__ bool get(int64_t u, int32_t& Jo, int32_t& Ko, int64_t& io) {
        if (tt < 0) return false;
        while (u >= base + cnt) {
            base += cnt;
            ++tt;
            if (!tiles.get(tt, J, K)) { tt = -1; return false; }
            cnt = pivots(J, K);
        }
        Jo = J;
        Ko = K;
        io = i_begin + (u - base);
        return true;
    }
};

__device__ __forceinline__ void ck_fold3(unsigned long long& lo, unsigned long long& hi,
                                         uint64_t l0, const uint32_t (&t)[8]) {
    uint64_t h = kCkSeed;
    h = fmix64(h ^ l0);
#pragma unroll
    for (int p = 0; p < 8; p += 2) h = fmix64(h ^ ((uint64_t)t[p] | ((uint64_t)t[p + 1] << 32)));
    uint64_t dlo = h, dhi = fmix64(h ^ kCkHi);
    unsigned long long nlo = lo + dlo;
    hi += dhi + (nlo < lo ? 1ull : 0ull);
    lo = nlo;
}

__device__ __forceinline__ void ck_flush3(unsigned long long lo, unsigned long long hi,
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

// bytewise a * b for a, b in {0,1,2} packed 4 per word: a*[b!=0] + a*[b==2].
__device__ __forceinline__ uint32_t mul_012(uint32_t a, uint32_t b) {
    const uint32_t nz = ((b | (b >> 1)) & 0x01010101u) * 0xFFu;
    const uint32_t two = ((b >> 1) & 0x01010101u) * 0xFFu;
    return (a & nz) + (a & two);
}

__device__ __forceinline__ int64_t c2(int64_t n) { return n * (n - 1) / 2; }
__device__ __forceinline__ int64_t c3(int64_t n) { return n * (n - 1) * (n - 2) / 6; }

__global__ void __launch_bounds__(kThreads3, 1)
tally3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const Tally3Args args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* smA = smem;
    uint8_t* smB = smem + kStages3 * kABytes3;
    uint8_t* smP = smem + kPivOff3;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBarOff3);
    uint64_t* xfull = full + kStages3;
    uint64_t* empty = xfull + kStages3;
    uint64_t* tfull = empty + kStages3;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < kStages3; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&xfull[s], 4);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpiWarps3);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    PivotSched sch;
    sch.init(args.n_v, args.i_begin, args.i_end);

    if (warp == 0) {
        if (lane == 0) {
            // ---------------------------------------------------------- TMA producer
            uint32_t stage = 0, phase = 0;
            const uint64_t pol = policy_evict_last();
            for (int64_t u = blockIdx.x;; u += gridDim.x) {
                int32_t J, K;
                int64_t i;
                if (!sch.get(u, J, K, i)) break;
                const int8_t* prow = args.N + i * args.k_pad;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], kABytes3 + kBBytes3 + kPivBytes);
                    tma_load_2d(smA + stage * kABytes3, &tmA, &full[stage], kb * kBK, J * kBM, pol);
                    tma_load_2d(smB + stage * kBBytes3, &tmB, &full[stage], kb * kBK, K * kBN, pol);
                    bulk_load(smP + stage * kPivBytes, prow + (int64_t)kb * kBK, kPivBytes,
                              &full[stage]);
                    if (++stage == kStages3) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------------------------------------------------- MMA issuer
            constexpr uint32_t idesc = idesc_i8(kBM, kBN);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            const uint32_t a0 = smem_u32(smA), b0 = smem_u32(smB);
            for (int64_t u = blockIdx.x;; u += gridDim.x) {
                int32_t J, K;
                int64_t i;
                if (!sch.get(u, J, K, i)) break;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * kBN;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait(&xfull[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = a0 + stage * kABytes3, sb = b0 + stage * kBBytes3;
#pragma unroll
                    for (int k = 0; k < kBK / kUMMA_K; ++k)
                        mma_i8(d, smem_desc_sw128(sa + k * kUMMA_K),
                               smem_desc_sw128(sb + k * kUMMA_K), idesc, (kb | k) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == kStages3) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp >= 2 + kEpiWarps3) {
        // -------------------------------------------------------------- transform
        const uint32_t r = (uint32_t)(warp - 2 - kEpiWarps3) * 32 + lane;  // tile row 0..127
        uint32_t stage = 0, phase = 0;
        for (int64_t u = blockIdx.x;; u += gridDim.x) {
            int32_t J, K;
            int64_t i;
            if (!sch.get(u, J, K, i)) break;
            for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                mbar_wait(&full[stage], phase);
                uint8_t* arow = smA + stage * kABytes3 + r * kBK;
                const uint8_t* pv = smP + stage * kPivBytes;
#pragma unroll
                for (uint32_t c = 0; c < 8; ++c) {
                    // 128-B swizzle: logical 16-B chunk c of row r sits at chunk c ^ (r & 7)
                    uint4* pa = reinterpret_cast<uint4*>(arow + ((c ^ (r & 7u)) << 4));
                    const uint4 y = *reinterpret_cast<const uint4*>(pv + (c << 4));
                    uint4 x = *pa;
                    x.x = mul_012(x.x, y.x);
                    x.y = mul_012(x.y, y.y);
                    x.z = mul_012(x.z, y.z);
                    x.w = mul_012(x.w, y.w);
                    *pa = x;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&xfull[stage]);
                if (++stage == kStages3) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // -------------------------------------------------------------- epilogue
        // Register-only drain (as in KB-2W): tcgen05.ld.16x256b gives a thread 2
        // consecutive k of 4 rows j; each triple record is 32 B of tallies + 64 B of fp64
        // CCC, i.e. whole L2 sectors written with 256-bit stores.
        // 8 warps: warp w drains lanes [half*16, half*16+16) of TMEM quadrant w % 4
        const uint32_t quad = warp & 3;
        const uint32_t half = (uint32_t)(warp - 2) >> 2;
        const int64_t n_v = args.n_v;
        const uint32_t fl = (uint32_t)args.out_flags;
        const bool want_t = fl & 1u, want_c64 = fl & 2u, want_c32 = fl & 4u, want_ck = fl & 8u;
        const bool want_c = want_c64 | want_c32;
        const uint32_t eight_nf = 8u * (uint32_t)args.n_f;
        const double inv8nf = 1.0 / (8.0 * (double)args.n_f);
        const int64_t c3n = c3(n_v);
        const int32_t cpair = 2 * (int32_t)(lane & 3);
        unsigned long long ck_lo = 0, ck_hi = 0;
        uint32_t acc = 0, acc_phase = 0;
        for (int64_t u = blockIdx.x;; u += gridDim.x) {
            int32_t J, K;
            int64_t i;
            if (!sch.get(u, J, K, i)) break;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t s_i = (uint32_t)__ldg(args.s + i);
            const double wi0 = __ldg(args.w + 2 * i) * inv8nf, wi1 = __ldg(args.w + 2 * i + 1) * inv8nf;
            // my 2 rows j = J*128 + quad*32 + half*16 + r*8 + lane/4
            int64_t rec_r[2], j_r[2];
            uint32_t s_j[2], g_ij[2];
            double wij[2][4];
            bool ok_r[2];
            bool my_any = false;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int64_t j = (int64_t)J * kBM + quad * 32 + half * 16 + r * 8 + (lane >> 2);
                j_r[r] = j;
                ok_r[r] = j > i && j < n_v;
                const int64_t jc = j < n_v ? j : n_v - 1;
                s_j[r] = (uint32_t)__ldg(args.s + jc);
                g_ij[r] = ok_r[r] ? (uint32_t)__ldg(args.G + i * n_v + j) : 0u;
                const double wj0 = __ldg(args.w + 2 * jc), wj1 = __ldg(args.w + 2 * jc + 1);
                wij[r][0] = wi0 * wj0;  // (a,b) = (0,0), includes 1/(8 n_f)
                wij[r][1] = wi0 * wj1;
                wij[r][2] = wi1 * wj0;
                wij[r][3] = wi1 * wj1;
                rec_r[r] = c3n - c3(n_v - i) + c2(n_v - i - 1) - c2(n_v - jc) - jc - 1 - args.rec_begin;
                my_any |= ok_r[r];
            }
            const bool any_row = __any_sync(0xffffffffu, my_any);
            const int64_t warp_jmin = __shfl_sync(0xffffffffu, j_r[0], 0);
            const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + acc * kBN;
            for (int c = 0; c < kBN / 8; ++c) {
                const int64_t k0 = (int64_t)K * kBN + c * 8;
                if (!any_row || k0 >= n_v || k0 + 8 <= warp_jmin + 1) continue;  // warp-uniform
                uint32_t va[4];
                tmem_ld_16x256(taddr + ((half * 16u) << 16) + c * 8, va);
                const int64_t kA = k0 + cpair, kB = kA + 1;
                const int64_t kAc = kA < n_v ? kA : n_v - 1, kBc = kB < n_v ? kB : n_v - 1;
                const uint32_t sA = (uint32_t)__ldg(args.s + kAc), sB = (uint32_t)__ldg(args.s + kBc);
                const uint32_t gikA = (uint32_t)__ldg(args.G + i * n_v + kAc);
                const uint32_t gikB = (uint32_t)__ldg(args.G + i * n_v + kBc);
                double wA0 = 0.0, wA1 = 0.0, wB0 = 0.0, wB1 = 0.0;
                if (want_c) {
                    wA0 = __ldg(args.w + 2 * kAc);
                    wA1 = __ldg(args.w + 2 * kAc + 1);
                    wB0 = __ldg(args.w + 2 * kBc);
                    wB1 = __ldg(args.w + 2 * kBc + 1);
                }
                tmem_ld_wait();
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if (!ok_r[r]) continue;
                    const int64_t j = j_r[r];
                    const uint32_t g3v[2] = {va[r * 2], va[r * 2 + 1]};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int64_t k = h ? kB : kA;
                        if (!(k > j && k < n_v)) continue;
                        const uint32_t g3 = g3v[h];
                        const uint32_t gij = g_ij[r], gik = h ? gikB : gikA;
                        const uint32_t gjk = (uint32_t)__ldg(args.G + j * n_v + k);
                        const uint32_t si = s_i, sj = s_j[r], sk = h ? sB : sA;
                        uint32_t t[8];   // Eq.5 cells, index 4a+2b+c, by inclusion-exclusion
                        t[7] = g3;                                       // (1,1,1)
                        t[6] = 2u * gij - g3;                            // (1,1,0)
                        t[5] = 2u * gik - g3;                            // (1,0,1)
                        t[3] = 2u * gjk - g3;                            // (0,1,1)
                        t[4] = 4u * si - 2u * gij - 2u * gik + g3;       // (1,0,0)
                        t[2] = 4u * sj - 2u * gij - 2u * gjk + g3;       // (0,1,0)
                        t[1] = 4u * sk - 2u * gik - 2u * gjk + g3;       // (0,0,1)
                        t[0] = eight_nf - 4u * (si + sj + sk) + 2u * (gij + gik + gjk) - g3;
                        const int64_t rec = rec_r[r] + k;
                        if (want_t)
                            stg_256_u32(args.tallies + 8 * rec, t[0], t[1], t[2], t[3], t[4], t[5],
                                        t[6], t[7]);
                        if (want_c) {
                            // Eq.4: CCC = T / (8 n_f) * w_i(a) w_j(b) w_k(c)
                            const double wk0 = h ? wB0 : wA0, wk1 = h ? wB1 : wA1;
                            double cc[8];
#pragma unroll
                            for (int ab = 0; ab < 4; ++ab) {
                                cc[2 * ab + 0] = (double)t[2 * ab + 0] * wij[r][ab] * wk0;
                                cc[2 * ab + 1] = (double)t[2 * ab + 1] * wij[r][ab] * wk1;
                            }
                            if (want_c64) {
                                double* p = reinterpret_cast<double*>(args.ccc) + 8 * rec;
                                stg_256_f64(p, cc[0], cc[1], cc[2], cc[3]);
                                stg_256_f64(p + 4, cc[4], cc[5], cc[6], cc[7]);
                            } else {
                                float* p = reinterpret_cast<float*>(args.ccc) + 8 * rec;
                                stg_256_u32(p, __float_as_uint((float)cc[0]), __float_as_uint((float)cc[1]),
                                            __float_as_uint((float)cc[2]), __float_as_uint((float)cc[3]),
                                            __float_as_uint((float)cc[4]), __float_as_uint((float)cc[5]),
                                            __float_as_uint((float)cc[6]), __float_as_uint((float)cc[7]));
                            }
                        }
                        if (want_ck)
                            ck_fold3(ck_lo, ck_hi,
                                     (3ull << 60) | ((uint64_t)i << 40) | ((uint64_t)j << 20) | (uint64_t)k, t);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (want_ck) ck_flush3(ck_lo, ck_hi, args.checksum);
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<512>(tmem_base);
}

cudaError_t launch_tally3(const CUtensorMap& tmA, const CUtensorMap& tmB, const Tally3Args& a,
                          int num_sms, cudaStream_t stream, int64_t* n_units_out) {
    PivotSched sch;
    sch.init(a.n_v, a.i_begin, a.i_end);
    int64_t units = 0;
    if (sch.tt >= 0) {
        TriSched t;
        t.init(0, a.n_v, a.n_v, 1);
        int32_t J, K;
        for (int64_t tt = 0; t.get(tt, J, K); ++tt) units += sch.pivots(J, K);
    }
    if (n_units_out) *n_units_out = units;
    if (units == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(tally3_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem3);
    if (e != cudaSuccess) return e;
    const int grid = (int)(units < num_sms ? units : num_sms);
    tally3_kernel<<<grid, kThreads3, kSmem3, stream>>>(tmA, tmB, a);
    return cudaGetLastError();
}

}  // namespace ccc
