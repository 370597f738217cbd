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
// The same holds for one block of the block-circulant decomposition (FsGeom: rows
// [a_lo, a_lo + nA) of block A against block B, the geometry of ccc_2way_block), which is
// how the field split composes with the vector-block ring into the paper's 2-D
// n_pv x n_pf grid: the tiles of that block's schedule are exported / owned.
// Slot layout per owner and wave [t_lo, t_hi): tile t (t mod world == owner) has slot
// q = (t - t_lo) / world; the partial of slice f sits at int32 offset
// ((q * world + f) << 16) + row * 256 + col (row < tile rows, col < 256).
// The finisher is HBM-bound: world * 4 B read + 48 B written per pair.
#include "sm100.cuh"
#include "common.cuh"
#include "internal.h"

#ifndef CCC_FS_MINB
#define CCC_FS_MINB 5   // CTAs per SM the register budget is fitted to
#endif

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
// (int2 slot loads; the two records' tallies leave as one 256-bit store).  The row terms
// (s_i, w_i(0) / 4n_f, w_i(1) / 4n_f) are computed once per tile into shared memory, so
// a thread carries only its column terms and kR x W partial loads in flight; W is the
// world size as a template constant (0 = runtime loop) so every load is issued before the
// first sum.  Register use stays low enough for 8+ CTAs per SM (the kernel is HBM-bound
// and needs the bytes in flight).
template <int W, bool CK>
__global__ void __launch_bounds__(128, CCC_FS_MINB) fs_finish_kernel(const int32_t* __restrict__ slots,
                                                        const int32_t* __restrict__ s_a,
                                                        const int32_t* __restrict__ s_b, FsGeom g,
                                                        int64_t n_f, double gamma, int32_t owner,
                                                        int32_t world_rt, int64_t t_lo, int64_t t_end,
                                                        int32_t tile_m, uint32_t flags,
                                                        uint32_t* __restrict__ tallies, void* ccc,
                                                        unsigned long long* checksum) {
    __shared__ double row_w0[256], row_w1[256];
    __shared__ uint32_t row_s[256];
    const int32_t world = W > 0 ? W : world_rt;
    TriSched sch;
    sch.init(g.a_lo, g.nA, g.nB, g.diag, tile_m, 2048, 2048);   // the schedule of ccc_2way_block
    const int64_t a_end = g.a_lo + g.nA, nB = g.nB;
    const int64_t rec_base = g.diag ? (g.a_lo * (2 * nB - g.a_lo - 1)) / 2 : 0;
    const int64_t first = t_lo + ((owner - t_lo % world) % world + world) % world;
    const int64_t owned = first < t_end ? (t_end - first + world - 1) / world : 0;
    const bool want_t = flags & 1u, want_c64 = flags & 2u, want_c32 = flags & 4u;
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
        __syncthreads();   // the previous tile's row terms are no longer read
        for (int r = threadIdx.x; r < tile_m; r += blockDim.x) {
            const int64_t i = g.a_lo + (int64_t)bm * tile_m + r;
            const uint32_t si = i < a_end ? (uint32_t)__ldg(s_a + i) : 0u;
            row_s[r] = si;
            row_w0[r] = (1.0 - gamma * ((two_nf - (double)si) / two_nf)) * inv4nf;
            row_w1[r] = (1.0 - gamma * ((double)si / two_nf)) * inv4nf;
        }
        __syncthreads();
        const int64_t j0 = (int64_t)bn * kBN + col;
        const bool ok0 = j0 < nB, ok1 = j0 + 1 < nB;
        const uint32_t sj0 = ok0 ? (uint32_t)__ldg(s_b + j0) : 0u;
        const uint32_t sj1 = ok1 ? (uint32_t)__ldg(s_b + j0 + 1) : 0u;
        const double wj00 = 1.0 - gamma * ((two_nf - (double)sj0) / two_nf);
        const double wj01 = 1.0 - gamma * ((double)sj0 / two_nf);
        const double wj10 = 1.0 - gamma * ((two_nf - (double)sj1) / two_nf);
        const double wj11 = 1.0 - gamma * ((double)sj1 / two_nf);
        const int64_t i0 = g.a_lo + (int64_t)bm * tile_m;
        // rows of this tile holding a record of column j0 or j0 + 1: i < a_end, and with
        // diag also i < j0 + 1 (A and B are one block, only i < j)
        int64_t r_end = (g.diag && j0 + 1 < a_end ? j0 + 1 : a_end) - i0;
        if (!ok0) r_end = 0;
        r_end = r_end < 0 ? 0 : (r_end > tile_m ? tile_m : r_end);
        constexpr int kR = W == 1 ? 8 : 4;   // rows in flight per thread
        for (int32_t row0 = 0; row0 < (int32_t)r_end; row0 += kR) {
            int2 Gr[kR];
#pragma unroll
            for (int u = 0; u < kR; ++u) Gr[u] = make_int2(0, 0);
            if constexpr (W > 0) {
                int2 v[kR][W];
#pragma unroll
                for (int u = 0; u < kR; ++u)
#pragma unroll
                    for (int f = 0; f < W; ++f)
                        v[u][f] = row0 + u < r_end
                                      ? __ldg(reinterpret_cast<const int2*>(tile + ((int64_t)f << 16) +
                                                                            (row0 + u) * kBN + col))
                                      : make_int2(0, 0);
#pragma unroll
                for (int u = 0; u < kR; ++u)
#pragma unroll
                    for (int f = 0; f < W; ++f) {
                        Gr[u].x += v[u][f].x;
                        Gr[u].y += v[u][f].y;
                    }
            } else {
                for (int32_t f = 0; f < world; ++f)
#pragma unroll
                    for (int u = 0; u < kR; ++u)
                        if (row0 + u < r_end) {
                            const int2 v = __ldg(reinterpret_cast<const int2*>(tile + ((int64_t)f << 16) +
                                                                               (row0 + u) * kBN + col));
                            Gr[u].x += v.x;
                            Gr[u].y += v.y;
                        }
            }
#pragma unroll
            for (int u = 0; u < kR; ++u) {
                const int32_t r = row0 + u;
                if (r >= r_end) break;
                const int64_t i = i0 + r;
                const uint32_t si = row_s[r];
                const double wi0 = row_w0[r], wi1 = row_w1[r];
                // diag: column j0 + 1 > i holds for every r < r_end
                const bool okA = !g.diag || j0 > i, okB = ok1;
                const uint32_t GA = (uint32_t)Gr[u].x, GB = (uint32_t)Gr[u].y;
                const uint32_t a3 = GA, a2 = 2u * si - GA, a1 = 2u * sj0 - GA, a0 = four_nf - 2u * si - 2u * sj0 + GA;
                const uint32_t b3 = GB, b2 = 2u * si - GB, b1 = 2u * sj1 - GB, b0 = four_nf - 2u * si - 2u * sj1 + GB;
                // record of column j0 (ccc_2way_block's layout)
                const int64_t rec = g.diag ? i * (2 * nB - i - 1) / 2 + (j0 - i - 1) - rec_base
                                           : (i - g.a_lo) * nB + j0;
                const uint64_t gi = (uint64_t)(g.a_row0 + i), gj = (uint64_t)(g.b_row0 + j0);
                if (want_t) {
                    if (okA && okB && !(rec & 1))
                        stg_256_u32(tallies + 4 * rec, a0, a1, a2, a3, b0, b1, b2, b3);
                    else {
                        if (okA) stg_128_u32(tallies + 4 * rec, a0, a1, a2, a3);
                        if (okB) stg_128_u32(tallies + 4 * (rec + 1), b0, b1, b2, b3);
                    }
                }
                if (want_c64) {
                    double* c = reinterpret_cast<double*>(ccc) + 4 * rec;
                    if (okA)
                        stg_256_f64(c, (double)a0 * wi0 * wj00, (double)a1 * wi0 * wj01, (double)a2 * wi1 * wj00,
                                    (double)a3 * wi1 * wj01);
                    if (okB)
                        stg_256_f64(c + 4, (double)b0 * wi0 * wj10, (double)b1 * wi0 * wj11,
                                    (double)b2 * wi1 * wj10, (double)b3 * wi1 * wj11);
                } else if (want_c32) {
                    float* c = reinterpret_cast<float*>(ccc) + 4 * rec;
                    if (okA)
                        stg_128_u32(c, __float_as_uint((float)((double)a0 * wi0 * wj00)),
                                    __float_as_uint((float)((double)a1 * wi0 * wj01)),
                                    __float_as_uint((float)((double)a2 * wi1 * wj00)),
                                    __float_as_uint((float)((double)a3 * wi1 * wj01)));
                    if (okB)
                        stg_128_u32(c + 4, __float_as_uint((float)((double)b0 * wi0 * wj10)),
                                    __float_as_uint((float)((double)b1 * wi0 * wj11)),
                                    __float_as_uint((float)((double)b2 * wi1 * wj10)),
                                    __float_as_uint((float)((double)b3 * wi1 * wj11)));
                }
                if constexpr (CK) {
                    if (okA)
                        fs_fold(ck_lo, ck_hi, (2ull << 60) | (gi << 40) | (gj << 20),
                                (uint64_t)a0 | ((uint64_t)a1 << 32), (uint64_t)a2 | ((uint64_t)a3 << 32));
                    if (okB)
                        fs_fold(ck_lo, ck_hi, (2ull << 60) | (gi << 40) | ((gj + 1) << 20),
                                (uint64_t)b0 | ((uint64_t)b1 << 32), (uint64_t)b2 | ((uint64_t)b3 << 32));
                }
            }
        }
    }
    if constexpr (CK) {
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

int64_t fs_block_tiles(const FsGeom& g) {
    TriSched sch;
    sch.init(g.a_lo, g.nA, g.nB, g.diag, tally2_tile_rows(), 2048, 2048);
    return sch.total();
}

int64_t fs_total_tiles(int64_t n_v) {
    FsGeom g{};
    g.nA = g.nB = n_v;
    g.diag = 1;
    return fs_block_tiles(g);
}

cudaError_t launch_fs_finish(const int32_t* slots, const int32_t* s_a, const int32_t* s_b, const FsGeom& g,
                             int64_t n_f, double gamma, int owner, int world, int64_t t_lo, int64_t t_hi,
                             uint32_t flags, uint32_t* tallies, void* ccc, unsigned long long* checksum,
                             int num_sms, cudaStream_t stream) {
    const int64_t all = fs_block_tiles(g);
    const int64_t t_end = (t_hi > 0 && t_hi < all) ? t_hi : all;
    if (t_end <= t_lo) return cudaSuccess;
    const int64_t owned = (t_end - t_lo + world - 1) / world;
    const bool ck = flags & 8u;
    auto go = [&](auto kern) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0) != cudaSuccess || per_sm < 1)
            per_sm = 4;
        const int64_t cap = (int64_t)per_sm * num_sms;
        const int64_t grid = owned < cap ? owned : cap;
        kern<<<(unsigned)grid, 128, 0, stream>>>(slots, s_a, s_b, g, n_f, gamma, owner, world, t_lo, t_end,
                                                 tally2_tile_rows(), flags, tallies, ccc, checksum);
    };
#define CCC_FS_CASE(w)                                                   \
    case w:                                                              \
        ck ? go(fs_finish_kernel<w, true>) : go(fs_finish_kernel<w, false>); \
        break;
    switch (world) {
        CCC_FS_CASE(1)
        CCC_FS_CASE(2)
        CCC_FS_CASE(3)
        CCC_FS_CASE(4)
        CCC_FS_CASE(8)
        default:
            ck ? go(fs_finish_kernel<0, true>) : go(fs_finish_kernel<0, false>);
    }
#undef CCC_FS_CASE
    return cudaGetLastError();
}

}  // namespace ccc
