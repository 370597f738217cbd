// tally3s.cu -- the sparse (missing-data) 3-way tally in ONE pass (
// PAPER.md §7 item 1; reading A-17).
//
// Method.  With n = allele-1 count (0 where the entry is missing) and v = [entry present],
// rho(1) = n and rho(0) = 2v - n, so every cell of the 3-way table is a signed combination
// of the eight trilinear forms
//     F[4 x_p + 2 x_m + x_n] = sum_q x_p x_m x_n,      x in {n (0), v (1)},
// namely T = (M (x) M (x) M) F with, per slot, allele 1 <- [n: 1, v: 0] and allele 0 <-
// [n: -1, v: 2]; c_pmn = F[7] (fields where all three are present) is the divisor:
// CCC(a,b,c) = T(a,b,c) / (8 c_pmn) w_p(a) w_m(b) w_n(c), 0 when c_pmn = 0.
//
// All eight forms of a (p, m, n) block come out of ONE tcgen05 GEMM: the operand is the
// group-interleaved X of the 2-way sparse mode (per 16 vectors: 16 rows n, then 16 rows v),
//   B = X rows of 128 n's (256 columns: per 32-column group 16 n's x {n, v}),
//   A = X rows of 64 m's (32 per CTA), each row weighted by the pivot's n_p AND by its
//       v_p (A o n_p and A o v_p stacked: 128 A rows per CTA),
// so the accumulator row (z, x_m, m) x column (x_n, n) holds F[4 z + 2 x_m + x_n] of the
// triple (p, m, n): 8 MACs per comparison, every form in TMEM at once, nothing stored in
// between (the first version ran 8 passes of the dense kernel and kept 7 forms in HBM).
//
// A row layout per CTA (128 rows = TMEM lanes): quadrant q = r / 32 holds m's 8q .. 8q+7
// of the CTA's 32; lane l = r % 32: z = l / 16, x_m = (l / 8) % 2, m = 8q + l % 8.  The
// transform warps build it from the TMA-staged 64 source rows (A-src ring) into the A ring.
// Epilogue: a warp drains its quadrant by 32-column groups (tcgen05.ld 32x32b.x16 twice:
// 16 n's x {n, v}); lane (g = 2z + x_m, m8) then holds one (z, x_m) combination of 16
// triples; a 4 x 4 transpose of 8-value blocks among the lanes {m8, m8+8, m8+16, m8+24}
// (3 shfl.xor rounds) gives each lane all 8 forms of 4 triples, which it turns into the 8
// tallies, CCC and 96 B (64 B with fp32 CCC) of records in the stage layout.
#include "sm100.cuh"
#include "common.cuh"
#include "internal.h"

namespace ccc {

namespace {

constexpr int kStS = 5;                     // pipeline stages
constexpr int kSrcBytes = 64 * kBK;         // 8 KB: 64 X rows (32 m's x {n, v}) per CTA
constexpr int kABytesS = 128 * kBK;         // 16 KB: the transformed A rows
constexpr int kBBytesS = 128 * kBK;         // 16 KB: this CTA's 128 B rows (64 n's x {n, v})
constexpr int kPivS = 2 * kBK;              // n_p and v_p chunks (128 B each)
constexpr int kEpiWarpsS = 8;
constexpr int kXfWarpsS = 4;
constexpr int kThreadsS = 32 * (2 + kEpiWarpsS + kXfWarpsS);
constexpr int kOffA = kStS * kSrcBytes;
constexpr int kOffB = kOffA + kStS * kABytesS;
constexpr int kOffP = kOffB + kStS * kBBytesS;
constexpr int kOffBar = kOffP + kStS * kPivS;
constexpr int kSmemS = kOffBar + 512 + 1024;
static_assert(kSmemS <= 232448, "sparse 3-way shared memory");
constexpr int kTileMs = 64;                 // m's per pair unit
constexpr int kTileNs = 128;                // n's per pair unit

__host__ __device__ __forceinline__ int64_t c2s(int64_t n) { return n * (n - 1) / 2; }
__host__ __device__ __forceinline__ int64_t c3s(int64_t n) { return n * (n - 1) * (n - 2) / 6; }

// Units (J, K, p): m-tile J (64 m's) x n-tile K (128 n's) with some m < n, pivots p in the
// stage's [p_lo, p_hi) with p < m and m < n possible; tiles J-major, pivots innermost so
// the concurrent CTA pairs share the tile's X rows in L2.
struct Sp3Sched {
    int64_t n_v, p_lo, p_hi;
    int32_t nJ, nK, J, K;
    int64_t base, cnt;
    bool done;
    __host__ __device__ int64_t pivots(int32_t j, int32_t k) const {
        int64_t m_max = (int64_t)j * kTileMs + kTileMs - 1;
        if (m_max > n_v - 1) m_max = n_v - 1;
        int64_t n_max = (int64_t)k * kTileNs + kTileNs - 1;
        if (n_max > n_v - 1) n_max = n_v - 1;
        int64_t hi = p_hi;
        if (hi > m_max) hi = m_max;            // p < m
        if (hi > n_max - 1) hi = n_max - 1;    // p < m < n
        return hi > p_lo ? hi - p_lo : 0;
    }
    __host__ __device__ bool next_tile() {   // advance (J, K) to the next tile in order
        if (++K >= nK) {
            ++J;
            if (J >= nJ) return false;
            K = J / 2;                         // first n-tile with an n above the tile's m's
        }
        return true;
    }
    __host__ __device__ void init(int64_t n_v_, int64_t p_lo_, int64_t p_hi_) {
        n_v = n_v_;
        p_lo = p_lo_;
        p_hi = p_hi_;
        nJ = (int32_t)((n_v + kTileMs - 1) / kTileMs);
        nK = (int32_t)((n_v + kTileNs - 1) / kTileNs);
        J = (int32_t)((p_lo + 1) / kTileMs);   // tiles whose m's all lie <= p_lo hold nothing
        K = J / 2;
        base = 0;
        done = J >= nJ;
        cnt = done ? 0 : pivots(J, K);
    }
    __host__ __device__ bool get(int64_t u, int32_t& Jo, int32_t& Ko, int64_t& po) {
        if (done) return false;
        while (u >= base + cnt) {
            base += cnt;
            if (!next_tile()) { done = true; return false; }
            cnt = pivots(J, K);
        }
        Jo = J;
        Ko = K;
        po = p_lo + (u - base);
        return true;
    }
};

__device__ __forceinline__ void ck_fold3s(unsigned long long& lo, unsigned long long& hi, uint64_t l0,
                                          const uint32_t (&t)[8]) {
    uint64_t h = kCkSeed;
    h = fmix64(h ^ l0);
#pragma unroll
    for (int p = 0; p < 8; p += 2) h = fmix64(h ^ ((uint64_t)t[p] | ((uint64_t)t[p + 1] << 32)));
    const uint64_t dlo = h, dhi = fmix64(h ^ kCkHi);
    const unsigned long long nlo = lo + dlo;
    hi += dhi + (nlo < lo ? 1ull : 0ull);
    lo = nlo;
}

struct Sp3Args {
    const int8_t* X;        // group-interleaved [rows][k_pad]
    const double* w;        // [n_v][2] sparse weights
    int64_t n_v, p_lo, p_hi, rec_base, k_pad;
    int32_t k_blocks, out_flags;
    uint32_t* tallies;
    void* ccc;
    unsigned long long* checksum;
};

__device__ __forceinline__ int64_t xrow(int64_t i, int x) { return 32 * (i >> 4) + 16 * x + (i & 15); }

}  // namespace

__global__ void __launch_bounds__(kThreadsS, 1)
tally3s_kernel(const __grid_constant__ CUtensorMap tmSrc, const __grid_constant__ CUtensorMap tmB,
               const Sp3Args args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* smS = smem;
    uint8_t* smA = smem + kOffA;
    uint8_t* smB = smem + kOffB;
    uint8_t* smP = smem + kOffP;
    uint64_t* aload = reinterpret_cast<uint64_t*>(smem + kOffBar);  // own A-src + pivots landed
    uint64_t* ready = aload + kStS;        // leader: both B halves + both transforms done
    uint64_t* empty = ready + kStS;        // both: the pair's MMAs consumed the stage
    uint64_t* tfull = empty + kStS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int64_t unit0 = blockIdx.x / 2, units = gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmSrc);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < kStS; ++s) {
            mbar_init(&aload[s], 1);
            mbar_init(&ready[s], 2 + 2 * kXfWarpsS);   // 2 producers + the pair's transform warps
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 2 * kEpiWarpsS);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t ready_leader = mapa_shared(smem_u32(&ready[0]), 0);
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), 0);

    Sp3Sched sch;
    sch.init(args.n_v, args.p_lo, args.p_hi);

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        uint32_t stage = 0, phase = 0;
        const uint64_t pol = policy_evict_last();
        for (int64_t u = unit0;; u += units) {
            int32_t J, K;
            int64_t p;
            if (!sch.get(u, J, K, p)) break;
            const int8_t* prow_n = args.X + xrow(p, 0) * args.k_pad;
            const int8_t* prow_v = args.X + xrow(p, 1) * args.k_pad;
            const int32_t srow = (int32_t)(2 * ((int64_t)J * kTileMs + rank * 32));   // X row of m-group
            const int32_t brow = (int32_t)(2 * (int64_t)K * kTileNs + rank * 128);
            for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                mbar_wait_sleep(&empty[stage], phase ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&aload[stage], kSrcBytes + kPivS);
                    tma_load_2d(smS + stage * kSrcBytes, &tmSrc, &aload[stage], kb * kBK, srow, pol);
                    bulk_load(smP + stage * kPivS, prow_n + (int64_t)kb * kBK, kBK, &aload[stage]);
                    bulk_load(smP + stage * kPivS + kBK, prow_v + (int64_t)kb * kBK, kBK, &aload[stage]);
                    const uint32_t rb = ready_leader + stage * 8u;
                    if (rank == 0) mbar_arrive_expect_tx(&ready[stage], 2 * kBBytesS);
                    else mbar_arrive_cluster(rb);
                    tma_load_2d_pair(smB + stage * kBBytesS, &tmB, rb, kb * kBK, brow, pol);
                }
                __syncwarp();
                if (++stage == kStS) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ------------------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = idesc_i8(256, kBN);
            uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
            const uint64_t a_desc0 = smem_desc_sw128(smem_u32(smA));
            const uint64_t b_desc0 = smem_desc_sw128(smem_u32(smB));
            for (int64_t u = unit0;; u += units) {
                int32_t J, K;
                int64_t p;
                if (!sch.get(u, J, K, p)) break;
                mbar_wait_sleep(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * kBN;
                for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                    mbar_wait_sleep(&ready[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = a_desc0 + ((stage * kABytesS) >> 4);
                    const uint64_t bd = b_desc0 + ((stage * kBBytesS) >> 4);
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < kBK / kUMMA_K; ++k)
                            mma_i8_pair(d, ad + (k * kUMMA_K >> 4), bd + (k * kUMMA_K >> 4), idesc, (kb | k) != 0);
                        mma_commit_pair(&empty[stage], 3);
                    }
                    __syncwarp();
                    if (++stage == kStS) { stage = 0; phase ^= 1; }
                }
                if (elect_one()) mma_commit_pair(&tfull[acc], 3);
                __syncwarp();
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp >= 2 + kEpiWarpsS) {
        // ------------------------------------------------------------------ transform
        // A row r (quadrant q = r/32, lane l = r%32: z = l/16, x_m = (l/8)%2, m = 8q + l%8)
        // <- source row 32 (m/16) + 16 x_m + m%16 of the staged X rows, times n_p (z = 0:
        // (a & [n_p >= 1]) + (a & [n_p == 2])) or v_p (z = 1: a & [v_p == 1]).  Thread
        // (q = transform warp, lane) owns chunk cl = lane % 8 of rows 32q + lane/8 + 4k,
        // k < 8: every warp access covers 4 whole 128-B rows (4 wavefronts, no conflicts).
        const uint32_t q = (uint32_t)(warp - 2 - kEpiWarpsS);
        const uint32_t cl = lane & 7u, a4 = lane >> 3;
        uint32_t stage = 0, phase = 0;
        for (int64_t u = unit0;; u += units) {
            int32_t J, K;
            int64_t p;
            if (!sch.get(u, J, K, p)) break;
            for (int32_t kb = 0; kb < args.k_blocks; ++kb) {
                mbar_wait_sleep(&aload[stage], phase);
                {
                    const uint4 pn = lds_v4(smP + stage * kPivS + cl * 16);
                    const uint4 pv = lds_v4(smP + stage * kPivS + kBK + cl * 16);
                    uint4 m1, m2, mv;
                    m1.x = ((pn.x | (pn.x >> 1)) & 0x01010101u) * 0xFFu;
                    m1.y = ((pn.y | (pn.y >> 1)) & 0x01010101u) * 0xFFu;
                    m1.z = ((pn.z | (pn.z >> 1)) & 0x01010101u) * 0xFFu;
                    m1.w = ((pn.w | (pn.w >> 1)) & 0x01010101u) * 0xFFu;
                    m2.x = ((pn.x >> 1) & 0x01010101u) * 0xFFu;
                    m2.y = ((pn.y >> 1) & 0x01010101u) * 0xFFu;
                    m2.z = ((pn.z >> 1) & 0x01010101u) * 0xFFu;
                    m2.w = ((pn.w >> 1) & 0x01010101u) * 0xFFu;
                    mv.x = (pv.x & 0x01010101u) * 0xFFu;
                    mv.y = (pv.y & 0x01010101u) * 0xFFu;
                    mv.z = (pv.z & 0x01010101u) * 0xFFu;
                    mv.w = (pv.w & 0x01010101u) * 0xFFu;
                    const uint8_t* src = smS + stage * kSrcBytes;
                    uint8_t* dst = smA + stage * kABytesS;
                    uint4 x[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t l = a4 + 4 * k;
                        const uint32_t m = 8 * q + (l & 7), xm = (l >> 3) & 1;
                        const uint32_t sr = 32 * (m >> 4) + 16 * xm + (m & 15);
                        x[k] = lds_v4(src + sr * kBK + ((cl ^ (sr & 7u)) << 4));
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t r = 32 * q + a4 + 4 * k;
                        if (k < 4) {   // z = n_p
                            x[k].x = (x[k].x & m1.x) + (x[k].x & m2.x);
                            x[k].y = (x[k].y & m1.y) + (x[k].y & m2.y);
                            x[k].z = (x[k].z & m1.z) + (x[k].z & m2.z);
                            x[k].w = (x[k].w & m1.w) + (x[k].w & m2.w);
                        } else {       // z = v_p
                            x[k].x &= mv.x;
                            x[k].y &= mv.y;
                            x[k].z &= mv.z;
                            x[k].w &= mv.w;
                        }
                        sts_v4(dst + r * kBK + ((cl ^ (r & 7u)) << 4), x[k].x, x[k].y, x[k].z, x[k].w);
                    }
                }
                __syncwarp();
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0) mbar_arrive(&ready[stage]);
                    else mbar_arrive_cluster(ready_leader + stage * 8u);
                }
                if (++stage == kStS) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // -------------------------------------------------------------------- epilogue
        const uint32_t q = warp & 3;                      // TMEM lane quadrant
        const uint32_t h = (uint32_t)(warp - 2) >> 2;     // column groups h, h+2, h+4, h+6
        const uint32_t g = lane >> 3, m8 = lane & 7;      // g = 2 z + x_m of my lane
        const uint32_t fl = (uint32_t)args.out_flags;
        const bool want_t = fl & 1u, want_c64 = fl & 2u, want_c32 = fl & 4u, want_ck = fl & 8u;
        const int64_t nv = args.n_v;
        unsigned long long ck_lo = 0, ck_hi = 0;
        uint32_t acc = 0, acc_phase = 0;
        for (int64_t u = unit0;; u += units) {
            int32_t J, K;
            int64_t p;
            if (!sch.get(u, J, K, p)) break;
            // my triples: m = J*64 + rank*32 + 8q + m8, n = K*128 + 16 cg + 4 g + jj
            const int64_t m = (int64_t)J * kTileMs + rank * 32 + 8 * q + m8;
            const bool m_ok = m > p && m < nv;
            const int64_t mc = m < nv ? m : nv - 1;
            const double wp0 = __ldg(args.w + 2 * p), wp1 = __ldg(args.w + 2 * p + 1);
            const double wm0 = __ldg(args.w + 2 * mc), wm1 = __ldg(args.w + 2 * mc + 1);
            const double wpm[4] = {wp0 * wm0, wp0 * wm1, wp1 * wm0, wp1 * wm1};   // [2 a_p + a_m]
            const int64_t rec_m = c3s(nv) - c3s(nv - p) + c2s(nv - p - 1) - c2s(nv - mc) - mc - 1 - args.rec_base;
            const bool any = __any_sync(0xffffffffu, m_ok);
            mbar_wait_sleep(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((q * 32u) << 16) + acc * kBN;
            for (int cgi = 0; cgi < 4 && any; ++cgi) {
                const int cg = (int)h + 2 * cgi;
                const int64_t n0 = (int64_t)K * kTileNs + 16 * cg;   // first n of the group
                if (n0 >= nv || n0 + 15 <= p + 1) continue;          // warp-uniform: nothing valid
                uint32_t v[32];
                tmem_ld16(taddr + cg * 32, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(taddr + cg * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld_wait();
                // blk[b][2 jj + x_n] = my F for n = n0 + 4 b + jj  (b = n block, jj < 4)
                uint32_t blk[4][8];
#pragma unroll
                for (int b = 0; b < 4; ++b)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        blk[b][2 * jj] = v[4 * b + jj];
                        blk[b][2 * jj + 1] = v[16 + 4 * b + jj];
                    }
                // 4 x 4 transpose of 8-value blocks among lanes m8 + 8 g': afterwards
                // F[g'][e] = lane (g', m8)'s value for my n block g (F[g][.] = my own)
                uint32_t F[4][8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    F[0][e] = g == 0 ? blk[0][e] : g == 1 ? blk[1][e] : g == 2 ? blk[2][e] : blk[3][e];
                }
#pragma unroll
                for (int d = 1; d < 4; ++d) {
                    const uint32_t gs = g ^ (uint32_t)d;   // the partner's block index
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const uint32_t send = gs == 0 ? blk[0][e] : gs == 1 ? blk[1][e] : gs == 2 ? blk[2][e] : blk[3][e];
                        F[d][e] = __shfl_xor_sync(0xffffffffu, send, 8 * d);
                    }
                }
                // F[d][.] came from lane g ^ d: reorder to G[g'] = forms of combination g'
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int64_t n = n0 + 4 * g + jj;
                    const bool ok = m_ok && n > m && n < nv;
                    uint32_t f8[8];   // f8[4 z + 2 x_m + x_n]
#pragma unroll
                    for (int gp = 0; gp < 4; ++gp) {
                        // combination gp sits in F[gp ^ g]
                        const uint32_t d = (uint32_t)gp ^ g;
                        const uint32_t a0 = d == 0 ? F[0][2 * jj] : d == 1 ? F[1][2 * jj] : d == 2 ? F[2][2 * jj] : F[3][2 * jj];
                        const uint32_t a1 = d == 0 ? F[0][2 * jj + 1] : d == 1 ? F[1][2 * jj + 1]
                                          : d == 2 ? F[2][2 * jj + 1] : F[3][2 * jj + 1];
                        f8[2 * gp] = a0;
                        f8[2 * gp + 1] = a1;
                    }
                    // T = (M x M x M) F, per slot: allele 1 <- n; allele 0 <- 2 v - n.
                    // slot n (x_n, the last index)
                    uint32_t s1[8];
#pragma unroll
                    for (int pm = 0; pm < 4; ++pm) {
                        s1[2 * pm + 1] = f8[2 * pm];                       // c = 1
                        s1[2 * pm] = 2u * f8[2 * pm + 1] - f8[2 * pm];     // c = 0
                    }
                    uint32_t s2[8];   // slot m
#pragma unroll
                    for (int pz = 0; pz < 2; ++pz)
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            s2[4 * pz + 2 + c] = s1[4 * pz + c];
                            s2[4 * pz + c] = 2u * s1[4 * pz + 2 + c] - s1[4 * pz + c];
                        }
                    uint32_t t[8];    // slot p: t[4 a + 2 b + c]
#pragma unroll
                    for (int bc = 0; bc < 4; ++bc) {
                        t[4 + bc] = s2[bc];
                        t[bc] = 2u * s2[4 + bc] - s2[bc];
                    }
                    const uint32_t cpmn = f8[7];
                    const int64_t rec = rec_m + n;
                    if (want_t)
                        stg_256_u32_if(ok, args.tallies + 8 * rec, t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
                    if (want_c64 || want_c32) {
                        const double inv = cpmn ? 1.0 / (8.0 * (double)cpmn) : 0.0;
                        const int64_t nc = n < nv ? n : nv - 1;
                        const double wn0 = __ldg(args.w + 2 * nc) * inv, wn1 = __ldg(args.w + 2 * nc + 1) * inv;
                        double cr[8];
#pragma unroll
                        for (int ab = 0; ab < 4; ++ab) {
                            cr[2 * ab] = u32_to_f64(t[2 * ab]) * wpm[ab] * wn0;
                            cr[2 * ab + 1] = u32_to_f64(t[2 * ab + 1]) * wpm[ab] * wn1;
                        }
                        if (want_c64) {
                            double* qd = reinterpret_cast<double*>(args.ccc) + 8 * rec;
                            stg_256_f64_if(ok, qd, cr[0], cr[1], cr[2], cr[3]);
                            stg_256_f64_if(ok, qd + 4, cr[4], cr[5], cr[6], cr[7]);
                        } else {
                            float* qf = reinterpret_cast<float*>(args.ccc) + 8 * rec;
                            stg_256_u32_if(ok, qf, __float_as_uint((float)cr[0]), __float_as_uint((float)cr[1]),
                                           __float_as_uint((float)cr[2]), __float_as_uint((float)cr[3]),
                                           __float_as_uint((float)cr[4]), __float_as_uint((float)cr[5]),
                                           __float_as_uint((float)cr[6]), __float_as_uint((float)cr[7]));
                        }
                    }
                    if (want_ck && ok)
                        ck_fold3s(ck_lo, ck_hi,
                                  (3ull << 60) | ((uint64_t)p << 40) | ((uint64_t)m << 20) | (uint64_t)n, t);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(tempty_leader + acc * 8u);
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (want_ck) {
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long olo = __shfl_xor_sync(0xffffffffu, ck_lo, o);
                const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, ck_hi, o);
                const unsigned long long nlo = ck_lo + olo;
                ck_hi += ohi + (nlo < ck_lo ? 1ull : 0ull);
                ck_lo = nlo;
            }
            if (lane == 0 && (ck_lo | ck_hi)) {
                const unsigned long long old = atomicAdd(&args.checksum[0], ck_lo);
                atomicAdd(&args.checksum[1], ck_hi + ((old + ck_lo < old) ? 1ull : 0ull));
            }
        }
    }

    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) tmem_dealloc_pair<512>(tmem_base);
}

int64_t sparse3_units(int64_t n_v, int64_t p_lo, int64_t p_hi) {
    Sp3Sched s;
    s.init(n_v, p_lo, p_hi);
    if (s.done) return 0;
    int64_t n = s.cnt;
    while (s.next_tile()) n += s.pivots(s.J, s.K);
    return n;
}

cudaError_t launch_tally3_sparse(const CUtensorMap& tmSrc, const CUtensorMap& tmB, const int8_t* X,
                                 const double* w, int64_t n_v, int64_t p_lo, int64_t p_hi, int64_t rec_base,
                                 int64_t k_pad, uint32_t out_flags, uint32_t* tallies, void* ccc,
                                 unsigned long long* checksum, int num_sms, cudaStream_t stream,
                                 int64_t* n_units_out) {
    const int64_t nu = sparse3_units(n_v, p_lo, p_hi);
    if (n_units_out) *n_units_out = nu;
    if (nu == 0) return cudaSuccess;
    Sp3Args a{};
    a.X = X;
    a.w = w;
    a.n_v = n_v;
    a.p_lo = p_lo;
    a.p_hi = p_hi;
    a.rec_base = rec_base;
    a.k_pad = k_pad;
    a.k_blocks = (int32_t)(k_pad / kBK);
    a.out_flags = (int32_t)out_flags;
    a.tallies = tallies;
    a.ccc = ccc;
    a.checksum = checksum;
    cudaError_t e = cudaFuncSetAttribute(tally3s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemS);
    if (e != cudaSuccess) return e;
    const int64_t pairs = num_sms / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * (nu < pairs ? nu : pairs)));
    cfg.blockDim = dim3(kThreadsS);
    cfg.dynamicSmemBytes = kSmemS;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, tally3s_kernel, tmSrc, tmB, a);
}

}  // namespace ccc
