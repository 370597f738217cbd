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
// so the TriSched cursor only walks forward); 128 threads, thread = 2 adjacent columns
// (int2 slot loads; the two records' tallies leave as one 256-bit store), 4 rows in flight.
__global__ void __launch_bounds__(128) fs_finish_kernel(const int32_t* __restrict__ slots,
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
    const int col = 2 * threadIdx.x;
    unsigned long long ck_lo = 0, ck_hi = 0;
    for (int64_t k = blockIdx.x; k < owned; k += gridDim.x) {
        const int64_t t = first + k * world;
        int32_t bm, bn;
        if (!sch.get(t, bm, bn)) break;
        const int64_t q = (t - t_lo) / world;
        const int32_t* tile = slots + ((q * world) << 16);
        int64_t j[2];
        bool col_ok[2];
        uint32_t sj[2];
        double wj0[2], wj1[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            j[h] = (int64_t)bn * kBN + col + h;
            col_ok[h] = j[h] < n_v;
            sj[h] = col_ok[h] ? (uint32_t)__ldg(s + j[h]) : 0u;
            wj0[h] = 1.0 - gamma * ((two_nf - (double)sj[h]) / two_nf);
            wj1[h] = 1.0 - gamma * ((double)sj[h] / two_nf);
        }
        constexpr int kR = 4;   // rows in flight per thread (memory-level parallelism)
        for (int32_t row0 = 0; row0 < tile_m; row0 += kR) {
            int2 Gr[kR];
#pragma unroll
            for (int u = 0; u < kR; ++u) {
                const int64_t i = (int64_t)bm * tile_m + row0 + u;
                Gr[u] = make_int2(0, 0);
                if (i < n_v - 1 && col_ok[0] && j[1] > i)
                    for (int32_t f = 0; f < world; ++f) {
                        const int2 v = __ldg(reinterpret_cast<const int2*>(tile + ((int64_t)f << 16) +
                                                                           (row0 + u) * kBN + col));
                        Gr[u].x += v.x;
                        Gr[u].y += v.y;
                    }
            }
#pragma unroll
            for (int u = 0; u < kR; ++u) {
                const int64_t i = (int64_t)bm * tile_m + row0 + u;
                if (i >= n_v - 1) continue;
                const uint32_t si = (uint32_t)__ldg(s + i);
                const double wi0 = (1.0 - gamma * ((two_nf - (double)si) / two_nf)) * inv4nf;
                const double wi1 = (1.0 - gamma * ((double)si / two_nf)) * inv4nf;
                uint32_t tt[2][4];
                double cc[2][4];
                bool ok[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    ok[h] = col_ok[h] && j[h] > i;
                    const uint32_t G = (uint32_t)(h ? Gr[u].y : Gr[u].x);
                    tt[h][3] = G;
                    tt[h][2] = 2u * si - G;
                    tt[h][1] = 2u * sj[h] - G;
                    tt[h][0] = four_nf - 2u * si - 2u * sj[h] + G;
                    cc[h][0] = (double)tt[h][0] * wi0 * wj0[h];
                    cc[h][1] = (double)tt[h][1] * wi0 * wj1[h];
                    cc[h][2] = (double)tt[h][2] * wi1 * wj0[h];
                    cc[h][3] = (double)tt[h][3] * wi1 * wj1[h];
                }
                const int64_t rec = i * (2 * n_v - i - 1) / 2 + (j[0] - i - 1);   // record of column col
                if (want_t) {
                    if (ok[0] && ok[1] && !(rec & 1))
                        stg_256_u32(tallies + 4 * rec, tt[0][0], tt[0][1], tt[0][2], tt[0][3], tt[1][0],
                                    tt[1][1], tt[1][2], tt[1][3]);
                    else
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            if (ok[h]) stg_128_u32(tallies + 4 * (rec + h), tt[h][0], tt[h][1], tt[h][2], tt[h][3]);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!ok[h]) continue;
                    if (want_c64)
                        stg_256_f64(reinterpret_cast<double*>(ccc) + 4 * (rec + h), cc[h][0], cc[h][1], cc[h][2],
                                    cc[h][3]);
                    else if (want_c32)
                        stg_128_u32(reinterpret_cast<float*>(ccc) + 4 * (rec + h), __float_as_uint((float)cc[h][0]),
                                    __float_as_uint((float)cc[h][1]), __float_as_uint((float)cc[h][2]),
                                    __float_as_uint((float)cc[h][3]));
                    if (want_ck)
                        fs_fold(ck_lo, ck_hi, (2ull << 60) | ((uint64_t)i << 40) | ((uint64_t)j[h] << 20),
                                (uint64_t)tt[h][0] | ((uint64_t)tt[h][1] << 32),
                                (uint64_t)tt[h][2] | ((uint64_t)tt[h][3] << 32));
                }
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
    fs_finish_kernel<<<(unsigned)grid, 128, 0, stream>>>(slots, s, n_v, n_f, gamma, owner, world, t_lo,
                                                         t_end, tally2_tile_rows(), flags, tallies, ccc,
                                                         checksum);
    return cudaGetLastError();
}

}  // namespace ccc
