// popcount.cu -- SURVEY §8(f) row f4(i): the paper's own tally method on B200's CUDA cores,
// kept as an on-device baseline for the tensor-core path (tally2.cu).
//
// The paper's mGEMM2 (§3.1) replaces the multiply-add of a GEMM by
// bitwise AND + population count over packed 2-bit genotypes.  Here the operands are the
// packed rows of ccc_pack themselves (16 codes per 32-bit word, code = (r1 << 1) | r2,
// P:259-268), and per word pair
//     sum_q n_iq n_jq = popc(x & y) + popc((xs & y) | ((x << 1) & y & H)),
// where n = r1 + r2, xs = (x >> 1) & 0x5555... moves r1 onto the r2 lane:
// (H = 0xAAAA...): popc(x & y) counts r1 r1' + r2 r2', the second term r1 r2' + r2 r1'.  With
// rho(0) = 2 - rho(1) the four tallies then follow from G and the row sums exactly as in
// the tensor-core path (Eq.2-3), so results are bit-identical.
//
// One CTA computes a 128 x 128 block of pairs (512 threads, 4 x 8 pairs each) on the
// upper block triangle; operand words are staged transposed in shared memory (16 words
// = 256 genotypes per step) together with their shifted forms, so a word pair costs
// 3 LOP + 2 POPC + 1 IADD: CUDA-core work at 8 comparisons per POPC.
#include "sm100.cuh"
#include "common.cuh"
#include "internal.h"

namespace ccc {

namespace {
constexpr int kPT = 128;        // pairs per tile side
constexpr int kPW = 16;         // packed words (x 16 genotypes) per shared-memory step
constexpr int kPS = kPT + 4;    // padded row: staging writes are 2-way instead of 16-way conflicts
constexpr uint32_t kLo = 0x55555555u;

__device__ __forceinline__ void pc_fold(unsigned long long& lo, unsigned long long& hi, uint64_t l0,
                                        uint64_t l1, uint64_t l2) {
    uint64_t h = kCkSeed;
    h = fmix64(h ^ l0);
    h = fmix64(h ^ l1);
    h = fmix64(h ^ l2);
    const uint64_t dlo = h, dhi = fmix64(h ^ kCkHi);
    const unsigned long long nlo = lo + dlo;
    hi += dhi + (nlo < lo ? 1ull : 0ull);
    lo = nlo;
}
}  // namespace

// s_i = sum_q (r1 + r2) = popcount of the packed row; w_i(a) = 1 - gamma f_i(a) (Eq.1).
__global__ void __launch_bounds__(256) popc_stats_kernel(const uint32_t* __restrict__ packed, int64_t n_v,
                                                         int64_t n_f, int64_t wpr, double gamma,
                                                         int32_t* __restrict__ s_out,
                                                         double* __restrict__ w_out) {
    const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (i >= n_v) return;
    const uint32_t* row = packed + i * wpr;
    int32_t s = 0;
    for (int64_t w = threadIdx.x & 31; w < wpr; w += 32) s += __popc(__ldg(row + w));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) {
        s_out[i] = s;
        const double two_nf = 2.0 * (double)n_f;
        w_out[2 * i + 0] = 1.0 - gamma * ((double)(2 * n_f - (int64_t)s) / two_nf);
        w_out[2 * i + 1] = 1.0 - gamma * ((double)s / two_nf);
    }
}

__global__ void __launch_bounds__(512, 1) popc_tally2_kernel(const uint32_t* __restrict__ packed, int64_t n_v,
                                                             int64_t n_f, int64_t wpr,
                                                             const int32_t* __restrict__ s,
                                                             const double* __restrict__ w, uint32_t flags,
                                                             uint32_t* __restrict__ tallies, void* ccc,
                                                             unsigned long long* checksum) {
    // per packed word, rows keep x, (x >> 1) & L and x << 1; columns keep y and y & H
    __shared__ __align__(16) uint32_t ra[kPW][kPS], rs[kPW][kPS], rl[kPW][kPS];
    __shared__ __align__(16) uint32_t cy[kPW][kPS], ch[kPW][kPS];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 8 columns x 4 rows per thread
    const int64_t nt = (n_v + kPT - 1) / kPT;
    const int64_t tiles = nt * (nt + 1) / 2;
    const bool want_t = flags & 1u, want_c64 = flags & 2u, want_c32 = flags & 4u, want_ck = flags & 8u;
    const double inv4nf = 1.0 / (4.0 * (double)n_f);
    const uint32_t four_nf = 4u * (uint32_t)n_f;
    unsigned long long ck_lo = 0, ck_hi = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        // tile t -> (I, J), I <= J, row-major over the upper block triangle
        int64_t I = 0, rem = t;
        while (rem >= nt - I) { rem -= nt - I; ++I; }
        const int64_t J = I + rem;
        const int64_t i0 = I * kPT, j0 = J * kPT;
        uint32_t g[4][8];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) g[a][b] = 0u;
        const uint32_t* prow = packed + i0 * wpr;
        const uint32_t* pcol = packed + j0 * wpr;
        const int nrow = (int)(n_v - i0 < kPT ? n_v - i0 : kPT);
        const int ncol = (int)(n_v - j0 < kPT ? n_v - j0 : kPT);
        for (int64_t w0 = 0; w0 < wpr; w0 += kPW) {
            __syncthreads();
            // stage 128 rows x 16 words of the row block and of the column block (transposed)
#pragma unroll
            for (int e = 0; e < (kPT * kPW) / 512; ++e) {
                const int idx = e * 512 + threadIdx.x;
                const int r = idx / kPW, k = idx % kPW;
                const bool okw = w0 + k < wpr;
                const uint32_t x = (r < nrow && okw) ? __ldg(prow + (int64_t)r * wpr + w0 + k) : 0u;
                const uint32_t y = (r < ncol && okw) ? __ldg(pcol + (int64_t)r * wpr + w0 + k) : 0u;
                ra[k][r] = x;
                rs[k][r] = (x >> 1) & kLo;
                rl[k][r] = x << 1;
                cy[k][r] = y;
                ch[k][r] = y & ~kLo;
            }
            __syncthreads();
#pragma unroll 2
            for (int k = 0; k < kPW; ++k) {
                uint32_t xa[4], xs[4], xl[4], yb[8], yh[8];
                *reinterpret_cast<uint4*>(xa) = *reinterpret_cast<const uint4*>(&ra[k][ty * 4]);
                *reinterpret_cast<uint4*>(xs) = *reinterpret_cast<const uint4*>(&rs[k][ty * 4]);
                *reinterpret_cast<uint4*>(xl) = *reinterpret_cast<const uint4*>(&rl[k][ty * 4]);
                *reinterpret_cast<uint4*>(&yb[0]) = *reinterpret_cast<const uint4*>(&cy[k][tx * 8]);
                *reinterpret_cast<uint4*>(&yb[4]) = *reinterpret_cast<const uint4*>(&cy[k][tx * 8 + 4]);
                *reinterpret_cast<uint4*>(&yh[0]) = *reinterpret_cast<const uint4*>(&ch[k][tx * 8]);
                *reinterpret_cast<uint4*>(&yh[4]) = *reinterpret_cast<const uint4*>(&ch[k][tx * 8 + 4]);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        // r1 r1' + r2 r2'  +  (r1 r2' at the r2 lane | r2 r1' at the r1 lane)
                        g[a][b] += __popc(xa[a] & yb[b]) + __popc((xs[a] & yb[b]) | (xl[a] & yh[b]));
            }
        }
        // epilogue: T11 = G, T10 = 2 s_i - G, T01 = 2 s_j - G, T00 = 4 n_f - 2 s_i - 2 s_j + G
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int64_t i = i0 + ty * 4 + a;
            if (i >= n_v) continue;
            const uint32_t si = (uint32_t)__ldg(s + i);
            const double wi0 = __ldg(w + 2 * i) * inv4nf, wi1 = __ldg(w + 2 * i + 1) * inv4nf;
            const int64_t rec_i = i * (2 * n_v - i - 1) / 2 - i - 1;   // p(i, j) = rec_i + j
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int64_t j = j0 + tx * 8 + b;
                if (j >= n_v || j <= i) continue;
                const uint32_t sj = (uint32_t)__ldg(s + j);
                const uint32_t G = g[a][b];
                const uint32_t t11 = G, t10 = 2u * si - G, t01 = 2u * sj - G;
                const uint32_t t00 = four_nf - 2u * si - 2u * sj + G;
                const int64_t rec = rec_i + j;
                if (want_t) stg_128_u32(tallies + 4 * rec, t00, t01, t10, t11);
                if (want_c64 || want_c32) {
                    const double wj0 = __ldg(w + 2 * j), wj1 = __ldg(w + 2 * j + 1);
                    const double c00 = (double)t00 * wi0 * wj0, c01 = (double)t01 * wi0 * wj1;
                    const double c10 = (double)t10 * wi1 * wj0, c11 = (double)t11 * wi1 * wj1;
                    if (want_c64)
                        stg_256_f64(reinterpret_cast<double*>(ccc) + 4 * rec, c00, c01, c10, c11);
                    else
                        stg_128_u32(reinterpret_cast<float*>(ccc) + 4 * rec, __float_as_uint((float)c00),
                                    __float_as_uint((float)c01), __float_as_uint((float)c10),
                                    __float_as_uint((float)c11));
                }
                if (want_ck)
                    pc_fold(ck_lo, ck_hi, (2ull << 60) | ((uint64_t)i << 40) | ((uint64_t)j << 20),
                            (uint64_t)t00 | ((uint64_t)t01 << 32), (uint64_t)t10 | ((uint64_t)t11 << 32));
            }
        }
    }
    if (want_ck) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long olo = __shfl_xor_sync(0xffffffffu, ck_lo, o);
            const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, ck_hi, o);
            const unsigned long long nlo = ck_lo + olo;
            ck_hi += ohi + (nlo < ck_lo ? 1ull : 0ull);
            ck_lo = nlo;
        }
        if ((threadIdx.x & 31) == 0 && (ck_lo | ck_hi)) {
            const unsigned long long old = atomicAdd(&checksum[0], ck_lo);
            atomicAdd(&checksum[1], ck_hi + ((old + ck_lo < old) ? 1ull : 0ull));
        }
    }
}

cudaError_t launch_popc_2way(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma, uint32_t flags,
                             uint32_t* tallies, void* ccc, unsigned long long* checksum, int32_t* s,
                             double* w, int num_sms, cudaStream_t stream) {
    const int64_t wpr = ((n_f + 63) / 64) * 4;   // packed row stride in 32-bit words
    const uint32_t* p = reinterpret_cast<const uint32_t*>(packed);
    popc_stats_kernel<<<(unsigned)((n_v + 7) / 8), 256, 0, stream>>>(p, n_v, n_f, wpr, gamma, s, w);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t nt = (n_v + kPT - 1) / kPT, tiles = nt * (nt + 1) / 2;
    const int64_t grid = tiles < 2 * (int64_t)num_sms ? tiles : 2 * (int64_t)num_sms;
    popc_tally2_kernel<<<(unsigned)grid, 512, 0, stream>>>(p, n_v, n_f, wpr, s, w, flags, tallies, ccc,
                                                          checksum);
    return cudaGetLastError();
}

}  // namespace ccc
