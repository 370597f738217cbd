// storebench.cu -- diagnostics: HBM write bandwidth of the store patterns an epilogue can use
// (what ceiling does the 3-way FULL output, 96 B per record, run into?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o storebench scripts/storebench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void stg256(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                       uint32_t f, uint32_t g, uint32_t h) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a), "r"(b), "r"(c),
                 "r"(d), "r"(e), "r"(f), "r"(g), "r"(h)
                 : "memory");
}

// mode 0: each warp instruction writes 1 KB contiguous (lane = 32-B record)
// mode 1: the 16x256b epilogue pattern: lane -> (row lane/4, records 2(lane%4) + h), rows 2 KB... apart
// mode 2: records of 96 B (32 B tally array + 64 B ccc array), mode-0 style (lane = record)
// mode 3: 96-B records in the 16x256b pattern (what tally3 does)
__global__ void __launch_bounds__(256) wr(uint8_t* T, uint8_t* C, int64_t recs, int mode, int64_t row_len) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const uint32_t v = lane;
    if (mode == 0 || mode == 2) {
        for (int64_t base = w0 * 32; base < recs; base += warps * 32) {
            const int64_t r = base + lane;
            if (r < recs) {
                stg256(T + 32 * r, v, v, v, v, v, v, v, v);
                if (mode == 2) {
                    stg256(C + 64 * r, v, v, v, v, v, v, v, v);
                    stg256(C + 64 * r + 32, v, v, v, v, v, v, v, v);
                }
            }
        }
    } else {
        // a "tile" = 16 rows x 8 records per warp step; rows are row_len records apart
        const int64_t per_tile = 16 * 8;
        const int64_t tiles = recs / per_tile;
        for (int64_t t = w0; t < tiles; t += warps) {
            const int64_t rows_per_band = row_len / 8;   // tiles per band of 16 rows
            const int64_t band = t / rows_per_band, colg = t % rows_per_band;
            for (int rr = 0; rr < 2; ++rr) {
                const int64_t row = band * 16 + rr * 8 + (lane >> 2);
                for (int h = 0; h < 2; ++h) {
                    const int64_t r = row * row_len + colg * 8 + 2 * (lane & 3) + h;
                    stg256(T + 32 * r, v, v, v, v, v, v, v, v);
                    if (mode == 3) {
                        stg256(C + 64 * r, v, v, v, v, v, v, v, v);
                        stg256(C + 64 * r + 32, v, v, v, v, v, v, v, v);
                    }
                }
            }
        }
    }
}

int main() {
    const int64_t recs = 1ll << 27;   // 134M records: 4 GB tallies + 8 GB ccc
    uint8_t *T, *C;
    cudaMalloc(&T, 32 * recs);
    cudaMalloc(&C, 64 * recs);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode)
        for (int cps : {1, 2, 4, 8})
            for (int64_t row_len : {256ll, 4096ll}) {
                if ((mode == 0 || mode == 2) && row_len != 256) continue;
                float best = 1e9;
                for (int it = 0; it < 4; ++it) {
                    cudaEventRecord(a);
                    wr<<<sms * cps, 256>>>(T, C, recs, mode, row_len);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (it > 0 && ms < best) best = ms;
                }
                const double bytes = (double)recs * ((mode >= 2) ? 96.0 : 32.0);
                printf("mode %d ctas/sm %d row_len %5lld: %.3f ms  %.0f GB/s\n", mode, cps,
                       (long long)row_len, best, bytes / best / 1e6);
            }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
