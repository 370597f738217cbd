// storebench2.cu -- diagnostics: how fast can W store warps per SM (one CTA per SM, like the
// 2-way epilogue) write 2-way FULL records (16 B tallies + 32 B fp64 CCC per pair) with
//   mode 0: the tally2 epilogue pattern from registers (lane -> row lane/4 (+8,+16,+24),
//           record pair 2(lane%4), 2(lane%4)+1 of an 8-column chunk; v8.b32 tallies,
//           2 x v4.f64 CCC per row), register values recomputed every chunk
//   mode 1: the same, CCC stores only
//   mode 2: the same, tally stores only
//   mode 3: records staged in shared memory, one cp.async.bulk (TMA) store per row segment
//           (CPC consecutive records of a row: CPC x 16 B tallies + CPC x 32 B CCC)
//   mode 4: contiguous 1 KB per warp store instruction (3 per chunk-row), the plain ceiling
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/storebench2 scripts/storebench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void stg_v8(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                       uint32_t f, uint32_t g, uint32_t h) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d),
                 "r"(e), "r"(f), "r"(g), "r"(h)
                 : "memory");
}
__device__ __forceinline__ void stg_f64x4(void* p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

template <int kMode, int kCPC>
__global__ void wr(uint32_t* T, double* C, int64_t rows, int64_t row_len, int chunks_per_warp) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * W + warp, nw = (int64_t)gridDim.x * W;
    const int64_t bands = rows / 32, cgs = row_len / kCPC;
    uint32_t seed = lane * 7u + 1u;
    uint8_t* stage = sm + (size_t)warp * 32 * kCPC * 48;   // 32 rows x kCPC records x 48 B
    for (int it = 0; it < chunks_per_warp; ++it) {
        const int64_t u = gw + (int64_t)it * nw;   // chunk id
        const int64_t band = (u / cgs) % bands, cg = u % cgs;
        const int64_t row0 = band * 32, col0 = cg * kCPC;
        seed = seed * 1664525u + 1013904223u;
        if constexpr (kMode <= 2) {
#pragma unroll
            for (int c8 = 0; c8 < kCPC / 8; ++c8) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int64_t row = row0 + r * 8 + (lane >> 2);
                    const int64_t rec = row * row_len + col0 + c8 * 8 + 2 * (lane & 3);
                    const uint32_t v = seed + r;
                    if (kMode != 1) stg_v8(T + 4 * rec, v, v + 1, v + 2, v + 3, v + 4, v + 5, v + 6, v + 7);
                    if (kMode != 2) {
                        const double d = (double)v;
                        stg_f64x4(C + 4 * rec, d, d + 1, d + 2, d + 3);
                        stg_f64x4(C + 4 * rec + 4, d + 4, d + 5, d + 6, d + 7);
                    }
                }
            }
        } else if constexpr (kMode == 3) {
            // stage: rows 0..31, tallies [32][kCPC][4] u32 then CCC [32][kCPC][4] f64
            uint32_t* st = reinterpret_cast<uint32_t*>(stage);
            double* sc = reinterpret_cast<double*>(stage + 32 * kCPC * 16);
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int c8 = 0; c8 < kCPC / 8; ++c8) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int row = r * 8 + (lane >> 2);
                    const int col = c8 * 8 + 2 * (lane & 3);
                    const uint32_t v = seed + r;
                    uint4* pt = reinterpret_cast<uint4*>(st + 4 * (row * kCPC + col));
                    pt[0] = make_uint4(v, v + 1, v + 2, v + 3);
                    pt[1] = make_uint4(v + 4, v + 5, v + 6, v + 7);
                    const double d = (double)v;
                    double2* pc = reinterpret_cast<double2*>(sc + 4 * (row * kCPC + col));
                    pc[0] = make_double2(d, d + 1);
                    pc[1] = make_double2(d + 2, d + 3);
                    pc[2] = make_double2(d + 4, d + 5);
                    pc[3] = make_double2(d + 6, d + 7);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            {
                const int row = lane;
                const int64_t rec = (row0 + row) * row_len + col0;
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(T + 4 * rec),
                             "r"(smem_u32(st + 4 * row * kCPC)), "r"(kCPC * 16)
                             : "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(C + 4 * rec),
                             "r"(smem_u32(sc + 4 * row * kCPC)), "r"(kCPC * 32)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        } else {
            // contiguous: the chunk's 32 x kCPC records as 3 x (32 x kCPC / 64) warp stores of 1 KB
            const int64_t rec0 = (row0 * row_len + col0 * 32);   // any disjoint region
            for (int k = 0; k < kCPC / 2; ++k) {
                const int64_t rec = rec0 + k * 64 + 2 * lane;
                const uint32_t v = seed + k;
                stg_v8(T + 4 * rec, v, v, v, v, v, v, v, v);
                stg_f64x4(C + 4 * rec, v, v, v, v);
                stg_f64x4(C + 4 * rec + 4, v, v, v, v);
            }
        }
    }
    if constexpr (kMode == 3) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int kMode, int kCPC>
void run(uint32_t* T, double* C, int sms, int W, int64_t rows, int64_t row_len) {
    const int64_t chunks = (rows / 32) * (row_len / kCPC);
    const int cpw = (int)(chunks / ((int64_t)sms * W));
    size_t smem = 200 * 1024;   // one CTA per SM
    if (kMode == 3 && (size_t)W * 32 * kCPC * 48 > smem) { printf("mode 3 W %d CPC %d: no smem\n", W, kCPC); return; }
    cudaFuncSetAttribute(wr<kMode, kCPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int i = 0; i < 5; ++i) {
        cudaEventRecord(a);
        wr<kMode, kCPC><<<sms, 32 * W, smem>>>(T, C, rows, row_len, cpw);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i > 0 && ms < best) best = ms;
    }
    const double recs = (double)cpw * sms * W * 32 * kCPC;
    const double bpr = kMode == 1 ? 32.0 : kMode == 2 ? 16.0 : 48.0;
    printf("mode %d CPC %2d warps/SM %2d: %.3f ms  %.0f GB/s  (%.2f B/clk/SM at 1.9 GHz)\n", kMode, kCPC, W, best,
           recs * bpr / best / 1e6, recs * bpr / (best * 1e-3) / sms / 1.9e9);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
    const int64_t rows = 20000 / 32 * 32, row_len = 10000;   // 2e8 records = 9.6 GB, like C2
    uint32_t* T;
    double* C;
    cudaMalloc(&T, (size_t)16 * rows * row_len);
    cudaMalloc(&C, (size_t)32 * rows * row_len);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int W : {4, 8, 16}) {
        run<0, 8>(T, C, sms, W, rows, row_len);
        run<1, 8>(T, C, sms, W, rows, row_len);
        run<2, 8>(T, C, sms, W, rows, row_len);
        run<4, 8>(T, C, sms, W, rows, row_len);
        run<3, 8>(T, C, sms, W, rows, row_len);
        run<3, 16>(T, C, sms, W, rows, row_len);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
