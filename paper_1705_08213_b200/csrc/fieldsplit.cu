// fieldsplit.cu -- SURVEY §8(f) row f3: the field-axis split (n_pf > 1, §4
// P:583-591), the one place where a collective FOLLOWS the tally GEMM.
//
// Each of `world` ranks holds all n_v vectors over a slice of the n_f fields and runs
// the tcgen05 tally GEMM (tally2.cu) on its slice in export mode: every partial tile
// G_f = N_f N_f^T leaves the epilogue straight into the slot of the tile's owner
// (owner(t) = t mod world) -- over NVLink through a peer-mapped pointer on a multi-GPU
// run -- while the tensor cores work on the next tiles.  That is the scatter half of a
// reduce-scatter, fused into the GEMM.  After a stream-ordered barrier, the owner's
// finishing kernel below reduces the `world` partials of each of its tiles (the reduce
// half: G = sum_f G_f, exact in int32) and applies the 2-way epilogue of Eq.2-3
// with the full allele sums s_i = sum_f s_i^f:
//     T11 = G, T10 = 2 s_i - G, T01 = 2 s_j - G, T00 = 4 n_f - 2 s_i - 2 s_j + G,
//     CCC(a,b) = T(a,b) / (4 n_f) w_i(a) w_j(b),  w(a) = 1 - gamma S(a) / (2 n_f)   (Eq.1).
// Slot layout per owner and wave [t_lo, t_hi): tile t (t mod world == owner) has slot
// q = (t - t_lo) / world; the partial of slice f sits at int32 offset
// ((q * world + f) << 16) + row * 256 + col (row < tile rows, col < 256).
// The finisher is HBM-bound: world * 4 B read + 48 B written per pair.
#include "sm100.cuh"
#include "common.cuh"
#include "internal.h"

namespace ccc {

namespace {
__device__ __forceinline__ void fs_fold(unsigned long long& lo, unsigned long long& hi, uint64_t l0,
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

// One CTA per owned tile at a time (tiles visited in increasing schedule order per CTA,
// so the TriSched cursor only walks forward); thread = column, loop over the tile rows.
__global__ void __launch_bounds__(256) fs_finish_kernel(const int32_t* __restrict__ slots,
                                                        const int32_t* __restrict__ s, int64_t n_v,
                                                        int64_t n_f, double gamma, int32_t owner,
                                                        int32_t world, int64_t t_lo, int64_t t_end,
                                                        int32_t tile_m, uint32_t flags,
                                                        uint32_t* __restrict__ tallies, void* ccc,
                                                        unsigned long long* checksum) {
    TriSched sch;
    sch.init(0, n_v, n_v, 1, tile_m, 2048, 2048);   // the schedule of ccc_2way_block(diag)
    const int64_t first = t_lo + ((owner - t_lo % world) % world + world) % world;
    const int64_t owned = first < t_end ? (t_end - first + world - 1) / world : 0;
    const bool want_t = flags & 1u, want_c64 = flags & 2u, want_c32 = flags & 4u, want_ck = flags & 8u;
    const double two_nf = 2.0 * (double)n_f, inv4nf = 1.0 / (4.0 * (double)n_f);
    const uint32_t four_nf = 4u * (uint32_t)n_f;
    const int col = threadIdx.x;
    unsigned long long ck_lo = 0, ck_hi = 0;
    for (int64_t k = blockIdx.x; k < owned; k += gridDim.x) {
        const int64_t t = first + k * world;
        int32_t bm, bn;
        if (!sch.get(t, bm, bn)) break;
        const int64_t q = (t - t_lo) / world;
        const int32_t* tile = slots + ((q * world) << 16);
        const int64_t j = (int64_t)bn * kBN + col;
        const bool col_ok = j < n_v;
        const uint32_t sj = col_ok ? (uint32_t)__ldg(s + j) : 0u;
        const double wj0 = 1.0 - gamma * ((two_nf - (double)sj) / two_nf);
        const double wj1 = 1.0 - gamma * ((double)sj / two_nf);
        constexpr int kR = 4;   // rows in flight per thread (memory-level parallelism)
        for (int32_t row0 = 0; row0 < tile_m; row0 += kR) {
          uint32_t Gr[kR];
#pragma unroll
          for (int u = 0; u < kR; ++u) {
            const int64_t i = (int64_t)bm * tile_m + row0 + u;
            Gr[u] = 0;
            if (i < n_v - 1 && col_ok && j > i)
                for (int32_t f = 0; f < world; ++f)
                    Gr[u] += (uint32_t)__ldg(tile + ((int64_t)f << 16) + (row0 + u) * kBN + col);
          }
#pragma unroll
          for (int u = 0; u < kR; ++u) {
            const int32_t row = row0 + u;
            const int64_t i = (int64_t)bm * tile_m + row;
            if (i >= n_v - 1 || !col_ok || j <= i) continue;
            const uint32_t G = Gr[u];
            const uint32_t si = (uint32_t)__ldg(s + i);
            const uint32_t t11 = G, t10 = 2u * si - G, t01 = 2u * sj - G;
            const uint32_t t00 = four_nf - 2u * si - 2u * sj + G;
            const int64_t rec = i * (2 * n_v - i - 1) / 2 + (j - i - 1);
            if (want_t) stg_128_u32(tallies + 4 * rec, t00, t01, t10, t11);
            if (want_c64 || want_c32) {
                const double wi0 = (1.0 - gamma * ((two_nf - (double)si) / two_nf)) * inv4nf;
                const double wi1 = (1.0 - gamma * ((double)si / two_nf)) * inv4nf;
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
                fs_fold(ck_lo, ck_hi, (2ull << 60) | ((uint64_t)i << 40) | ((uint64_t)j << 20),
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

int64_t fs_total_tiles(int64_t n_v) {
    TriSched sch;
    sch.init(0, n_v, n_v, 1, tally2_tile_rows(), 2048, 2048);
    return sch.total();
}

cudaError_t launch_fs_finish(const int32_t* slots, const int32_t* s, int64_t n_v, int64_t n_f, double gamma,
                             int owner, int world, int64_t t_lo, int64_t t_hi, uint32_t flags,
                             uint32_t* tallies, void* ccc, unsigned long long* checksum, int num_sms,
                             cudaStream_t stream) {
    const int64_t all = fs_total_tiles(n_v);
    const int64_t t_end = (t_hi > 0 && t_hi < all) ? t_hi : all;
    if (t_end <= t_lo) return cudaSuccess;
    const int64_t owned = (t_end - t_lo + world - 1) / world;
    const int64_t grid = owned < 8 * (int64_t)num_sms ? owned : 8 * (int64_t)num_sms;
    fs_finish_kernel<<<(unsigned)grid, 256, 0, stream>>>(slots, s, n_v, n_f, gamma, owner, world, t_lo,
                                                         t_end, tally2_tile_rows(), flags, tallies, ccc,
                                                         checksum);
    return cudaGetLastError();
}

}  // namespace ccc
