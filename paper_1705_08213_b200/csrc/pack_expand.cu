// pack_expand.cu -- KB-pack and KB-expand. HBM-bound.
//
// pack  : one byte per genotype code -> 2 bits per code, 4 codes per byte, LSB
//         first, rows padded to 64-entry (16-byte) units -- the storage density of
//         the paper's packed double-complex word.
// expand: packed codes -> int8 allele-1 counts n_{iq} = rho_{i,q}(1)
//         laid out K-major with rows padded to K_pad = 128-byte multiples (zero pad:
//         padding contributes nothing to N N^T, so no correction term is needed,
//         cf. P:444-446), plus the per-vector sums s_i = S_i(1) and the frequency
//         weights w_i(a) = 1 - gamma f_i(a) of Eq.1/Eq.3.
#include "common.cuh"
#include "internal.h"

namespace ccc {

__device__ __forceinline__ uint32_t pack16(const uint4 c) {
    const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
    uint32_t out = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        uint32_t x = cw[b] & 0x03030303u;  // 4 codes, one per byte
        // gather bits: byte k (2 bits) -> bits 2k..2k+1
        x = (x | (x >> 6)) & 0x000F000Fu;
        x = (x | (x >> 12)) & 0xFFu;
        out |= x << (8 * b);
    }
    return out;
}

// Warp per vector row (8 rows per CTA in flight, grid-stride over rows).  A warp pass
// covers 128 packed words: lane l handles words base + 32 u + l (u = 0..3), so each of the
// four 16-B code loads and each 4-B word store of the pass is one contiguous warp access,
// with four loads in flight per lane.  A warp per row keeps the ragged end of a row to a
// fraction of one warp pass (a CTA per row left up to 255 threads idle on the last pass).
__device__ __forceinline__ uint32_t pack_word_scalar(const uint8_t* row, int64_t n_f, int64_t g) {
    uint32_t out = 0;
    const int64_t q0 = g * 16;
    for (int u = 0; u < 16; ++u) {
        const int64_t q = q0 + u;
        if (q < n_f) out |= (uint32_t)(row[q] & 3u) << (2 * u);
    }
    return out;
}

__global__ void __launch_bounds__(256) pack_kernel(const uint8_t* __restrict__ codes,
                                                   int64_t n_v, int64_t n_f, int64_t words_per_row,
                                                   uint32_t* __restrict__ packed) {
    // rows are 16-B aligned when n_f % 16 == 0 (uint4 loads), 4-B aligned when n_f % 4 == 0
    // (four u32 loads per word, e.g. the field slices of f3); otherwise bytes
    const uintptr_t base_addr = reinterpret_cast<uintptr_t>(codes);
    const bool vec16 = (n_f % 16) == 0 && (base_addr % 16) == 0;
    const bool vec4 = !vec16 && (n_f % 4) == 0 && (base_addr % 4) == 0;
    const int64_t full = (vec16 || vec4) ? n_f / 16 : 0;   // words made of 16 in-range codes
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n_v; i += (int64_t)gridDim.x * 8) {
        const uint8_t* row = codes + i * n_f;
        uint32_t* prow = packed + i * words_per_row;
        const uint4* crow = reinterpret_cast<const uint4*>(row);
        const uint32_t* crow4 = reinterpret_cast<const uint32_t*>(row);
        auto load16 = [&](int64_t g) -> uint4 {
            if (vec16) return __ldcs(crow + g);
            return make_uint4(__ldcs(crow4 + 4 * g), __ldcs(crow4 + 4 * g + 1), __ldcs(crow4 + 4 * g + 2),
                              __ldcs(crow4 + 4 * g + 3));
        };
        int64_t base = 0;
        for (; base + 128 <= full; base += 128) {
            uint4 c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) c[u] = load16(base + 32 * u + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) prow[base + 32 * u + lane] = pack16(c[u]);
        }
        for (int64_t g = base + lane; g < words_per_row; g += 32)
            prow[g] = g < full ? pack16(load16(g)) : pack_word_scalar(row, n_f, g);
    }
}

// Warp per vector row (8 rows per CTA): a warp pass covers 128 packed words, lane l words
// base + 32 u + l -> four coalesced 4-B loads in flight, four coalesced 16-B streaming
// stores of int8 counts; the row sum is a warp reduction (no CTA barrier between rows).
__device__ __forceinline__ uint4 expand_word(uint32_t p) {
    // n = r1 + r2 per 2-bit code: (p & 0x5555...) + ((p >> 1) & 0x5555...)
    const uint32_t cnt = (p & 0x55555555u) + ((p >> 1) & 0x55555555u);
    uint32_t o[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        uint32_t x = (cnt >> (8 * b)) & 0xFFu;  // 4 counts, 2 bits each
        x = (x | (x << 12)) & 0x000F000Fu;
        x = (x | (x << 6)) & 0x03030303u;
        o[b] = x;
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

__global__ void __launch_bounds__(256) expand_kernel(const uint32_t* __restrict__ packed,
                                                     int64_t n_v, int64_t n_f,
                                                     int64_t words_per_row, int64_t k_pad,
                                                     double gamma, int8_t* __restrict__ N,
                                                     int32_t* __restrict__ s_out,
                                                     double* __restrict__ w_out) {
    const int64_t groups = k_pad / 16;   // output words (16 counts each), a multiple of 8
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n_v; i += (int64_t)gridDim.x * 8) {
        const uint32_t* prow = packed + i * words_per_row;
        uint4* nrow = reinterpret_cast<uint4*>(N + i * k_pad);
        int32_t sum = 0;
        for (int64_t base = 0; base < groups; base += 128) {
            uint32_t p[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t g = base + 32 * u + lane;
                p[u] = g < words_per_row ? __ldg(prow + g) : 0u;
                // codes past n_f in the last word are not elements (whatever the caller's
                // padding holds): mask them like expand_sparse_kernel does
                const int64_t left = n_f - 16 * g;
                if (left < 16) p[u] &= left <= 0 ? 0u : (uint32_t)((1ull << (2 * left)) - 1);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t g = base + 32 * u + lane;
                sum += __popc(p[u]);   // sum of r1 + r2 over the 16 codes
                if (g < groups) __stcs(nrow + g, expand_word(p[u]));
            }
        }
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        if (lane == 0) {
            s_out[i] = sum;
            const double two_nf = 2.0 * (double)n_f;
            const double f1 = (double)sum / two_nf;                       // Eq.1, a = 1
            const double f0 = (double)(2 * n_f - (int64_t)sum) / two_nf;  // Eq.1, a = 0
            w_out[2 * i + 0] = 1.0 - gamma * f0;
            w_out[2 * i + 1] = 1.0 - gamma * f1;
        }
    }
}

// Single-GPU fused form of pack + expand: unpacked codes (one byte each, 0..3) straight to
// the int8 operand N, s and w -- the same outputs as expand_kernel on ccc_pack's output,
// in one HBM pass (1 B read + 1 B written per element instead of 1 + 0.25 + 0.25 + 1).
// The 2-bit packed form is what crosses NVLink in the multi-GPU ring; a single GPU whose
// input arrives unpacked never needs it.  Warp per vector row, warp passes of 128 output
// words (16 counts each): lane l handles words base + 32 u + l, four 16-B code loads in
// flight, four coalesced 16-B streaming stores; n = r1 + r2 per byte, s = popcount of the
// 2-bit codes (the same as popcount of the packed word).
__device__ __forceinline__ uint32_t count4(uint32_t c) {
    c &= 0x03030303u;                                   // 4 codes, one per byte
    return (c & 0x01010101u) + ((c >> 1) & 0x01010101u);
}

__device__ __forceinline__ uint4 codes16_tail(const uint8_t* row, int64_t n_f, int64_t g) {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    for (int u = 0; u < 16; ++u) {
        const int64_t q = g * 16 + u;
        if (q < n_f) w[u >> 2] |= (uint32_t)row[q] << (8 * (u & 3));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(256) expand_codes_kernel(const uint8_t* __restrict__ codes, int64_t n_v,
                                                           int64_t n_f, int64_t k_pad, double gamma,
                                                           int8_t* __restrict__ N, int32_t* __restrict__ s_out,
                                                           double* __restrict__ w_out) {
    const uintptr_t base_addr = reinterpret_cast<uintptr_t>(codes);
    const bool vec16 = (n_f % 16) == 0 && (base_addr % 16) == 0;
    const bool vec4 = !vec16 && (n_f % 4) == 0 && (base_addr % 4) == 0;
    const int64_t full = (vec16 || vec4) ? n_f / 16 : 0;   // output words of 16 in-range codes
    const int64_t groups = k_pad / 16;
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n_v; i += (int64_t)gridDim.x * 8) {
        const uint8_t* row = codes + i * n_f;
        const uint4* crow = reinterpret_cast<const uint4*>(row);
        const uint32_t* crow4 = reinterpret_cast<const uint32_t*>(row);
        uint4* nrow = reinterpret_cast<uint4*>(N + i * k_pad);
        auto load16 = [&](int64_t g) -> uint4 {
            if (vec16) return __ldcs(crow + g);
            return make_uint4(__ldcs(crow4 + 4 * g), __ldcs(crow4 + 4 * g + 1), __ldcs(crow4 + 4 * g + 2),
                              __ldcs(crow4 + 4 * g + 3));
        };
        auto emit = [&](int64_t g, uint4 c, int32_t& sum) {
            const uint4 n = make_uint4(count4(c.x), count4(c.y), count4(c.z), count4(c.w));
            sum += __popc(c.x & 0x03030303u) + __popc(c.y & 0x03030303u) + __popc(c.z & 0x03030303u) +
                   __popc(c.w & 0x03030303u);
            __stcs(nrow + g, n);
        };
        int32_t sum = 0;
        int64_t base = 0;
        for (; base + 128 <= full; base += 128) {
            uint4 c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) c[u] = load16(base + 32 * u + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) emit(base + 32 * u + lane, c[u], sum);
        }
        for (int64_t g = base + lane; g < groups; g += 32)
            emit(g, g < full ? load16(g) : codes16_tail(row, n_f, g), sum);
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        if (lane == 0) {
            s_out[i] = sum;
            const double two_nf = 2.0 * (double)n_f;
            const double f1 = (double)sum / two_nf;                       // Eq.1, a = 1
            const double f0 = (double)(2 * n_f - (int64_t)sum) / two_nf;  // Eq.1, a = 0
            w_out[2 * i + 0] = 1.0 - gamma * f0;
            w_out[2 * i + 1] = 1.0 - gamma * f1;
        }
    }
}

// Sparse (missing-data) mode, §7 item 1, reading A-17: the code
// (1,0) marks a missing entry.  One warp per vector i writes two operand rows of the
// group-interleaved matrix X (groups of 16 vectors: 16 rows n, then 16 rows v):
//   X[32 (i/16) + i%16]      = n_{iq} = rho_{i,q}(1) on present entries, 0 if missing
//   X[32 (i/16) + 16 + i%16] = v_{iq} = [entry present], 0 on the K padding
// and s_i = sum of n, c_i = #present, w_i(a) = 1 - gamma S_i(a) / (2 c_i) (1 if c_i = 0).
// Rows of the padding vectors n_v <= i < n_v16 are written as zeros.
__global__ void __launch_bounds__(256) expand_sparse_kernel(
    const uint32_t* __restrict__ packed, int64_t n_v, int64_t n_v16, int64_t n_f,
    int64_t words_per_row, int64_t k_pad, double gamma, int8_t* __restrict__ X,
    int32_t* __restrict__ s_out, int32_t* __restrict__ c_out, double* __restrict__ w_out) {
    // X is the operand of both sparse modes (2-way tally2, 3-way tally3s)
    // a warp per vector (8 per CTA), warp passes of 128 packed words as in expand_kernel
    const int64_t groups = k_pad / 16;
    const int lane = threadIdx.x & 31;
    for (int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); i < n_v16; i += (int64_t)gridDim.x * 8) {
        const bool real = i < n_v;
        const uint32_t* prow = packed + i * words_per_row;
        const int64_t xr = 32 * (i / 16) + (i % 16);
        uint4* nrow = reinterpret_cast<uint4*>(X + xr * k_pad);
        uint4* vrow = reinterpret_cast<uint4*>(X + (xr + 16) * k_pad);
        int32_t sum = 0, cnt = 0;
        for (int64_t base = 0; base < groups; base += 128) {
            uint32_t pw[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t g = base + 32 * u + lane;
                pw[u] = (real && g < words_per_row) ? __ldg(prow + g) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t g = base + 32 * u + lane;
                if (g >= groups) continue;
                const uint32_t p = pw[u];
                const int64_t left = n_f - 16 * g;       // codes of this group inside n_f
                const uint32_t inside = !real || left <= 0 ? 0u
                                        : left >= 16 ? 0x55555555u
                                                     : (uint32_t)((1ull << (2 * left)) - 1) & 0x55555555u;
                const uint32_t lo = p & 0x55555555u, hi = (p >> 1) & 0x55555555u;   // r2, r1
                const uint32_t present = (~hi | lo) & inside;       // not (r1, r2) = (1, 0)
                const uint32_t n = lo + (hi & lo);                   // r1 + r2 if present, else 0
                uint32_t on[4], ov[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    uint32_t x = (n >> (8 * b)) & 0xFFu;
                    x = (x | (x << 12)) & 0x000F000Fu;
                    on[b] = (x | (x << 6)) & 0x03030303u;
                    uint32_t y = (present >> (8 * b)) & 0xFFu;
                    y = (y | (y << 12)) & 0x000F000Fu;
                    ov[b] = (y | (y << 6)) & 0x03030303u;
                }
                sum += __popc(lo) + __popc(hi & lo);
                cnt += __popc(present);
                __stcs(nrow + g, make_uint4(on[0], on[1], on[2], on[3]));
                __stcs(vrow + g, make_uint4(ov[0], ov[1], ov[2], ov[3]));
            }
        }
        for (int off = 16; off > 0; off >>= 1) {
            sum += __shfl_xor_sync(0xffffffffu, sum, off);
            cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        }
        if (lane == 0 && real) {
            s_out[i] = sum;
            c_out[i] = cnt;
            const double two_c = 2.0 * (double)cnt;
            const double f1 = cnt ? (double)sum / two_c : 0.0;                 // S_i(1) / (2 c_i)
            const double f0 = cnt ? (double)(2 * cnt - sum) / two_c : 0.0;     // S_i(0) / (2 c_i)
            w_out[2 * i + 0] = 1.0 - gamma * f0;
            w_out[2 * i + 1] = 1.0 - gamma * f1;
        }
    }
}

cudaError_t launch_expand_sparse(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma,
                                 int8_t* X, int32_t* s, int32_t* c, double* w, int num_sms,
                                 cudaStream_t stream) {
    const int64_t wpr = (n_f + 63) / 64 * 4;
    const int64_t k_pad = (n_f + 127) / 128 * 128;
    const int64_t n_v16 = (n_v + 15) / 16 * 16;
    const int64_t rows_blocks = (n_v16 + 7) / 8;   // a warp per row, 8 per CTA
    int64_t blocks = rows_blocks < (int64_t)num_sms * 8 ? rows_blocks : (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    expand_sparse_kernel<<<(int)blocks, 256, 0, stream>>>(
        reinterpret_cast<const uint32_t*>(packed), n_v, n_v16, n_f, wpr, k_pad, gamma, X, s, c, w);
    return cudaGetLastError();
}


// f4(ii), the paper's 3-way route (Table 1, P:457-516 with reading A-3): one int8 mask row
// per class xi of the pivot's genotype -- xi = 1: (0,0), xi = 2: heterozygote, xi = 3:
// (1,1) -- over the true n_f fields (K padding and tail are 0), plus the class counts.
__global__ void __launch_bounds__(256) expand_masks_kernel(const uint32_t* __restrict__ packed, int64_t n_v,
                                                           int64_t n_f, int64_t words_per_row, int64_t k_pad,
                                                           int8_t* __restrict__ M, int32_t* __restrict__ cnt) {
    __shared__ int32_t red[3][8];
    const int64_t groups = k_pad / 16;
    const size_t mat = (size_t)n_v * (size_t)k_pad;
    for (int64_t i = blockIdx.x; i < n_v; i += gridDim.x) {
        const uint32_t* prow = packed + i * words_per_row;
        int32_t c[3] = {0, 0, 0};
        for (int64_t g = threadIdx.x; g < groups; g += blockDim.x) {
            const uint32_t p = g < words_per_row ? __ldg(prow + g) : 0u;
            const int64_t left = n_f - 16 * g;
            const uint32_t inside = left <= 0 ? 0u : left >= 16 ? 0x55555555u
                                                                : (uint32_t)((1ull << (2 * left)) - 1) & 0x55555555u;
            const uint32_t lo = p & 0x55555555u, hi = (p >> 1) & 0x55555555u;
            const uint32_t cls[3] = {~(lo | hi) & inside, (lo ^ hi) & inside, lo & hi & inside};
#pragma unroll
            for (int x = 0; x < 3; ++x) {
                uint32_t o[4];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    uint32_t y = (cls[x] >> (8 * b)) & 0xFFu;
                    y = (y | (y << 12)) & 0x000F000Fu;
                    o[b] = (y | (y << 6)) & 0x03030303u;
                }
                c[x] += __popc(cls[x]);
                __stcs(reinterpret_cast<uint4*>(M + x * mat + i * k_pad) + g, make_uint4(o[0], o[1], o[2], o[3]));
            }
        }
#pragma unroll
        for (int x = 0; x < 3; ++x)
            for (int off = 16; off > 0; off >>= 1) c[x] += __shfl_xor_sync(0xffffffffu, c[x], off);
        if ((threadIdx.x & 31) == 0)
            for (int x = 0; x < 3; ++x) red[x][threadIdx.x >> 5] = c[x];
        __syncthreads();
        if (threadIdx.x < 3) {
            int32_t v = 0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) v += red[threadIdx.x][k];
            cnt[threadIdx.x * n_v + i] = v;
        }
        __syncthreads();
    }
}

cudaError_t launch_expand_masks(const uint8_t* packed, int64_t n_v, int64_t n_f, int8_t* M, int32_t* cnt,
                                int num_sms, cudaStream_t stream) {
    const int64_t wpr = (n_f + 63) / 64 * 4;
    const int64_t k_pad = (n_f + 127) / 128 * 128;
    int64_t blocks = n_v < (int64_t)num_sms * 8 ? n_v : (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    expand_masks_kernel<<<(int)blocks, 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(packed), n_v, n_f,
                                                         wpr, k_pad, M, cnt);
    return cudaGetLastError();
}

cudaError_t launch_pack(const uint8_t* codes, int64_t n_v, int64_t n_f, uint8_t* packed,
                        int num_sms, cudaStream_t stream) {
    const int64_t wpr = (n_f + 63) / 64 * 4;
    const int64_t rows_blocks = (n_v + 7) / 8;   // a warp per row, 8 per CTA
    int64_t blocks = rows_blocks < (int64_t)num_sms * 8 ? rows_blocks : (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    pack_kernel<<<(int)blocks, 256, 0, stream>>>(codes, n_v, n_f, wpr,
                                                 reinterpret_cast<uint32_t*>(packed));
    return cudaGetLastError();
}

cudaError_t launch_expand(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma,
                          int8_t* N, int32_t* s, double* w, int num_sms, cudaStream_t stream) {
    const int64_t wpr = (n_f + 63) / 64 * 4;
    const int64_t k_pad = (n_f + 127) / 128 * 128;
    const int64_t rows_blocks = (n_v + 7) / 8;   // a warp per row, 8 per CTA
    int64_t blocks = rows_blocks < (int64_t)num_sms * 8 ? rows_blocks : (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    expand_kernel<<<(int)blocks, 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(packed),
                                                   n_v, n_f, wpr, k_pad, gamma, N, s, w);
    return cudaGetLastError();
}

cudaError_t launch_expand_codes(const uint8_t* codes, int64_t n_v, int64_t n_f, double gamma, int8_t* N,
                                int32_t* s, double* w, int num_sms, cudaStream_t stream) {
    const int64_t k_pad = (n_f + 127) / 128 * 128;
    const int64_t rows_blocks = (n_v + 7) / 8;   // a warp per row, 8 per CTA
    int64_t blocks = rows_blocks < (int64_t)num_sms * 8 ? rows_blocks : (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    expand_codes_kernel<<<(int)blocks, 256, 0, stream>>>(codes, n_v, n_f, k_pad, gamma, N, s, w);
    return cudaGetLastError();
}

}  // namespace ccc
