/*
 * ccc.h -- C ABI of libccc, the B200 (sm_100a) CCC tally engine.
 *
 * Implements the hot path of PAPER.md (arXiv 1705.08213, "Parallel Accelerated
 * Custom Correlation Coefficient Calculations for Genomics Applications"): for n_v
 * vectors of n_f 2-bit genotype entries, the 2x2 (2-way) / 2x2x2 (3-way) allele
 * co-occurrence tallies of every unique pair i<j / triple i<j<k and the CCC values
 * formed from them and the per-vector allele frequencies.
 *
 *   v_{i,q} = (r1, r2) in S_2                                  P:259-264 (§2.1)
 *   rho_{i,q}(a) = #{r in v_{i,q} : r = a}
 *   f_i(a)   = (1/2n_f) sum_q rho_{i,q}(a)                       Eq.1
 *   f_ij(a,b) = (1/4n_f) sum_q rho_{i,q}(a) rho_{j,q}(b)         Eq.2
 *   CCC_ij(a,b) = f_ij(a,b)(1 - g f_i(a))(1 - g f_j(b)), g=2/3   Eq.3
 *   f_ijk(a,b,c) = (1/8n_f) sum_q rho_i(a) rho_j(b) rho_k(c)     Eq.5
 *   CCC_ijk = f_ijk (1-g f_i(a))(1-g f_j(b))(1-g f_k(c))          Eq.4
 *   unique results: distinct i<j, i<j<k
 *
 * CONVENTIONS (all functions)
 *  - Element code: one byte code = 2*r1 + r2 in {0,1,2,3}; (1,0) and (0,1) are the
 *    same heterozygote in dense mode.  Indices are 0-based.
 *  - Tally cell order is a-major: [T00,T01,T10,T11] and [T000 ... T111] with slot
 *    order (i,j,k) as in Eq.5.  Tallies are integer counts (sum = 4n_f / 8n_f);
 *    f = T/(4n_f) or T/(8n_f).  CCC is computed in fp64 (or emitted as fp32).
 *  - Records are emitted in lexicographic order of (i,j) / (i,j,k); see
 *    ccc_pair_index / ccc_triple_index.
 *  - Pointers named *_d are DEVICE pointers (CUDA global memory of the current
 *    device), *_h HOST pointers.  The caller owns every buffer; the library never
 *    allocates, frees or retains caller memory.  Scratch comes from a caller
 *    workspace sized by ccc_workspace_bytes.  No hidden global state besides a
 *    thread-local error string and a per-process device-property cache.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device functions only enqueue work: they are asynchronous on `stream`;
 *    execution faults surface at the caller's next synchronisation.
 *  - Arguments are validated synchronously before any launch.  Invalid sizes or
 *    NULL / misaligned (16 B) required pointers -> CCC_ERR_INVALID_ARGUMENT; a
 *    device that is not sm_100 -> CCC_ERR_UNSUPPORTED; n_f > CCC_MAX_NF (int32
 *    accumulator bound 8 n_f < 2^31) -> CCC_ERR_UNSUPPORTED; a launch failure ->
 *    CCC_ERR_CUDA with detail in ccc_last_error().  n_v < num_way is not an error:
 *    the result is empty and nothing is launched.
 *  - Re-entrant; calls on different streams / devices may run concurrently.
 */
#ifndef CCC_H_
#define CCC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CCC_OK = 0,
    CCC_ERR_INVALID_ARGUMENT = 1,
    CCC_ERR_UNSUPPORTED = 2,
    CCC_ERR_CUDA = 3,
    CCC_ERR_WORKSPACE = 4
} ccc_status;

/* Output selection bits (out_flags). */
enum {
    CCC_OUT_TALLY = 1,     /* uint32 tallies [records][4 or 8]                         */
    CCC_OUT_CCC_F64 = 2,   /* double CCC     [records][4 or 8]                         */
    CCC_OUT_CCC_F32 = 4,   /* float  CCC     [records][4 or 8] (exclusive with F64)    */
    CCC_OUT_CHECKSUM = 8   /* add every record's 128-bit digest into checksum_d[2]      */
};

#define CCC_MAX_NF 268435455LL   /* 8 * n_f must fit an int32 TMEM accumulator      */
#define CCC_MAX_NV 1048575LL     /* 20-bit index fields of the checksum digest       */

/* ---------------------------------------------------------------- host helpers */

/* Library / ABI version (major*10000 + minor*100 + patch). */
int ccc_version(void);

/* Human-readable name of a status code (static storage). */
const char* ccc_status_string(int status);

/* Detail of the last error raised on the calling thread ("" if none). */
const char* ccc_last_error(void);

/* Number of unique results: C(n_v,2) for num_way=2, C(n_v,3) for num_way=3
 * (P:293-295); 0 when n_v < num_way; -1 for an invalid num_way. */
int64_t ccc_num_unique(int num_way, int64_t n_v);

/* Lexicographic record index of pair i<j: i(2n_v-i-1)/2 + (j-i-1); -1 if not
 * 0 <= i < j < n_v. */
int64_t ccc_pair_index(int64_t n_v, int64_t i, int64_t j);

/* Lexicographic record index of triple i<j<k:
 * C(n_v,3) - C(n_v-i,3) + C(n_v-i-1,2) - C(n_v-j,2) + (k-j-1); -1 if invalid. */
int64_t ccc_triple_index(int64_t n_v, int64_t i, int64_t j, int64_t k);

/* Byte stride of one packed vector: ceil(n_f/64)*16 (64 entries per 16 bytes, the
 * density of the paper's double-complex packing unit). */
int64_t ccc_packed_stride(int64_t n_f);

/* Byte stride of one row of the expanded allele-count matrix N: ceil(n_f/128)*128. */
int64_t ccc_k_pad(int64_t n_f);

/* 3-way stages: stage s of n_stages covers pivots i in [i_begin,i_end)
 * (first index of the triple), i.e. the contiguous record range
 * [rec_begin, rec_begin+rec_count) of the lexicographic triple array.  Boundaries
 * balance the record count.  out[4] = {i_begin, i_end, rec_begin, rec_count}. */
ccc_status ccc_stage_range(int64_t n_v, int64_t n_stages, int64_t stage, int64_t* out);

/* Device workspace bytes needed by ccc_2way (num_way=2) or ccc_3way_prepare /
 * ccc_3way_stage / ccc_3way (num_way=3) for this problem size. */
size_t ccc_workspace_bytes(int num_way, int64_t n_v, int64_t n_f);

/* ---------------------------------------------------------------- device path */

/* KB-pack (§8(a) a1; P:403-410 packing): codes_d uint8 [n_v][n_f] (row-major, one
 * code per byte, values 0..3; higher bits are ignored) -> packed_d uint8
 * [n_v][ccc_packed_stride(n_f)], element q of vector i in bits 2(q%4)..2(q%4)+1 of
 * byte q/4 of its row (LSB first); the tail of each row is zero. */
ccc_status ccc_pack(const uint8_t* codes_d, int64_t n_v, int64_t n_f, uint8_t* packed_d,
                    void* stream);

/* Threshold-compacted output ("very few of the elements
 * are actually needed -- only those above a certain threshold").  Passed as the
 * `compact` argument of ccc_2way, ccc_2way_block, ccc_3way_stage, ccc_3way_unit and
 * ccc_3way; NULL selects the dense record layout.  When non-NULL, a record is kept iff
 * the largest of its 4 (8) CCC cells is > threshold (computed in fp64 whatever the
 * output precision), and every kept record is appended at an arbitrary free slot:
 *   keys_d[slot]    = i * 2^20 + j (2-way) or i * 2^40 + j * 2^20 + k (3-way), GLOBAL
 *                     indices, i < j < k
 *   tallies_d[slot] = its 4 (8) tallies (if CCC_OUT_TALLY), ccc_d[slot] = its CCC cells
 *                     (if CCC_OUT_CCC_F64 / _F32), both [capacity][cells]
 * *count_d (zeroed by the caller; accumulates across calls) is increased by the number
 * of kept records.  If it ends above `capacity`, only `capacity` of the kept records
 * (an arbitrary subset) were stored: re-run with a larger buffer.  The checksum, if
 * requested, still covers every record.  Slot order is nondeterministic. */
typedef struct {
    double threshold;
    int64_t capacity;     /* records keys_d / tallies_d / ccc_d can hold */
    uint64_t* keys_d;     /* [capacity], 8-B aligned (device) */
    uint64_t* count_d;    /* one counter (device), 8-B aligned */
} ccc_compact;

/* KB-expand (§8(a) a2; Eq.1): packed_d -> N_d int8 [n_v][ccc_k_pad(n_f)] with
 * N[i][q] = rho_{i,q}(1) in {0,1,2} (0 for q >= n_f), s_d int32 [n_v] with
 * s_i = sum_q rho_{i,q}(1) = S_i(1), and w_d double [n_v][2] with
 * w_i(a) = 1 - gamma * f_i(a), f_i(1) = s_i/(2n_f), f_i(0) = (2n_f - s_i)/(2n_f).
 * N_d must be 128-B aligned. */
ccc_status ccc_expand(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                      int8_t* N_d, int32_t* s_d, double* w_d, void* stream);

/* KB-expand straight from unpacked codes (§8(a) a1+a2 fused for a single GPU; Eq.1,
 * P:270-278): codes_d uint8 [n_v][n_f] (row-major, code = 2 r1 + r2, only the low 2 bits
 * of each byte are read) -> the same N_d / s_d / w_d as ccc_pack followed by ccc_expand,
 * in one HBM pass.  The 2-bit packed form exists for storage and for the
 * multi-GPU ring, where it is what crosses NVLink; one GPU fed unpacked codes skips it.
 * N_d 128-B aligned; errors as ccc_expand. */
ccc_status ccc_expand_codes(const uint8_t* codes_d, int64_t n_v, int64_t n_f, double gamma,
                            int8_t* N_d, int32_t* s_d, double* w_d, void* stream);

/* Whole 2-way problem on one GPU (§8(a) a2-a4): expand packed_d into the workspace,
 * then the persistent tcgen05 kind::i8 tally GEMM G = N N^T over the upper
 * triangle with the fused epilogue
 *   T11 = G, T10 = 2s_i - G, T01 = 2s_j - G, T00 = 4n_f - 2s_i - 2s_j + G,
 *   CCC(a,b) = T(a,b) / (4n_f) * w_i(a) * w_j(b)                   (Eq.2-3)
 * writing record p = ccc_pair_index(n_v,i,j) for every i<j:
 *   tallies_d uint32 [C(n_v,2)][4]   (if out_flags & CCC_OUT_TALLY)
 *   ccc_d     double/float [C(n_v,2)][4] (CCC_OUT_CCC_F64 / _F32)
 *   checksum_d uint64 [2] (lo, hi) += sum of record digests (CCC_OUT_CHECKSUM; the
 *              caller zeroes it first).
 * Outputs not selected may be NULL.  ws_d: >= ccc_workspace_bytes(2,...) bytes,
 * 256-B aligned.  compact: NULL, or the threshold-compacted layout (ccc_compact). */
ccc_status ccc_2way(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                    uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                    void* ws_d, size_t ws_bytes, const ccc_compact* compact, void* stream);

/* The same whole 2-way problem from UNPACKED device codes (§8(a) a1-a4 on one GPU; the
 * bench's step): codes_d uint8 [n_v][n_f] (row-major, code = 2 r1 + r2, low 2 bits read)
 * -> ccc_expand_codes into the workspace (one HBM pass, no 2-bit intermediate), then the
 * fused tally GEMM + epilogue of ccc_2way.  ws_d >= ccc_workspace_bytes(2, n_v, n_f),
 * 256-B aligned; outputs, flags, compaction and errors as ccc_2way. */
ccc_status ccc_2way_codes(const uint8_t* codes_d, int64_t n_v, int64_t n_f, double gamma,
                          uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                          void* ws_d, size_t ws_bytes, const ccc_compact* compact, void* stream);

/* The paper's own 2-way tally method on CUDA cores (§3.1
 * mGEMM2): the same problem and outputs as ccc_2way, computed from the
 * packed 2-bit rows with bitwise AND + population count instead of tensor-core MACs,
 *   G_ij = sum_w popc(x & y) + popc((xs & y) | ((x & ys) << 1)),  xs = (x >> 1) & 0x55..,
 * then the Eq.2-3 epilogue of ccc_2way (general-gamma form: CCC = T * (w_i(a)/(4n_f)) *
 * w_j(b) with w from Eq.1).  An on-device comparison baseline, not the product path.
 * packed_d as produced by ccc_pack; ws_d >= ccc_workspace_bytes(2, n_v, n_f) bytes,
 * 256-B aligned (only the s / w part is used); other arguments and errors as ccc_2way
 * (no compaction). */
ccc_status ccc_2way_popcount(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                             uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                             uint64_t* checksum_d, void* ws_d, size_t ws_bytes, void* stream);

/* ---- f3: field-axis split with the reduce-scatter fused onto the GEMM (
 * PAPER.md §4: n_pf > 1 processors share the fields of every vector).
 * `world` ranks each hold all n_v vectors over a slice of the fields (any split; each
 * slice is packed / expanded on its own with its own n_f_slice).  Per wave of tiles
 * [t_lo, t_hi) of the 2-way schedule (0 <= t_lo <= t_hi <= ccc_2way_fs_tiles(n_v)):
 *   1. every rank: ccc_2way_fs_export -- the tcgen05 tally GEMM of its slice; each
 *      partial tile G_f = N_f N_f^T is stored by the GEMM epilogue straight into the
 *      slot buffer of the tile's owner (owner(t) = t mod world), i.e. over NVLink when
 *      slots_d[owner] is a peer mapping (ccc_ipc_*), overlapped with later tiles;
 *   2. a stream-ordered barrier across ranks (the caller's, e.g. an NCCL all-reduce);
 *   3. every rank r: ccc_2way_fs_finish -- sums the `world` partials of its own tiles
 *      (exact int32) and writes their records exactly as ccc_2way (Eq.2-3), with the
 *      full allele sums s_d (the caller sums the slices' s, e.g. all-reduce) and the full
 *      n_f; general-gamma CCC form, w(a) = 1 - gamma S(a)/(2 n_f) computed inline.
 * Slot buffer of one owner: ccc_2way_fs_slot_bytes(world, t_lo, t_hi) bytes (int32
 * [owned tiles][world][256][256]); slots_d: DEVICE array of `world` device pointers (the
 * owners' buffers as this rank sees them).  A slot buffer may be reused by a later wave
 * once every owner's finish of the earlier wave is ordered before the new exports.
 * Records of a rank's own tiles only are written (tallies/ccc/checksum as ccc_2way;
 * per-rank checksums add up mod 2^128 to ccc_2way's). */
#define CCC_IPC_HANDLE_BYTES 64
int64_t    ccc_2way_fs_tiles(int64_t n_v);
size_t     ccc_2way_fs_slot_bytes(int world, int64_t t_lo, int64_t t_hi);
ccc_status ccc_2way_fs_export(const int8_t* N_d, const int32_t* s_d, int64_t n_v, int64_t n_f_slice,
                              int32_t* const* slots_d, int rank, int world, int64_t t_lo, int64_t t_hi,
                              void* stream);
ccc_status ccc_2way_fs_finish(const int32_t* slots_d, const int32_t* s_d, int64_t n_v, int64_t n_f,
                              double gamma, int rank, int world, int64_t t_lo, int64_t t_hi,
                              uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                              void* stream);
/* The same fused reduce-scatter for ONE block of the block-circulant decomposition -- the
 * composition of the field split with the vector-block ring, i.e. the paper's 2-D
 * n_pv x n_pf grid: the ranks of one field group each hold the same
 * two vector blocks A, B over their own field slice and split the tiles of the block's
 * schedule among themselves (owner(t) = t mod world).  Geometry exactly as
 * ccc_2way_block: rows [a_lo, a_hi) of block A (n_a rows, global row 0 = a_row0) against
 * the n_b rows of block B (b_row0); diag != 0: A and B are one block (same pointers,
 * n_a == n_b) and only local pairs i < j.  Tiles: ccc_2way_fs_block_tiles (-1 on invalid
 * geometry); slot sizing and the wave protocol as above.  Export: N_a / N_b int8
 * [rows][ccc_k_pad(n_f_slice)] (128-B aligned) and the slice's s_a / s_b (read only by the
 * per-row setup).  Finish: s_a / s_b = the FULL allele sums of the two blocks (s_a == s_b
 * when diag), n_f = the full field count; records land in ccc_2way_block's layout for
 * that geometry (own tiles only), checksum keys use the global indices.  Errors as
 * ccc_2way_fs_export / ccc_2way_fs_finish. */
int64_t    ccc_2way_fs_block_tiles(int64_t n_a, int64_t a_lo, int64_t a_hi, int64_t n_b, int diag);
ccc_status ccc_2way_fs_block_export(const int8_t* N_a, const int32_t* s_a, int64_t n_a, int64_t a_lo,
                                    int64_t a_hi, const int8_t* N_b, const int32_t* s_b, int64_t n_b,
                                    int diag, int64_t n_f_slice, int32_t* const* slots_d, int rank,
                                    int world, int64_t t_lo, int64_t t_hi, void* stream);
ccc_status ccc_2way_fs_block_finish(const int32_t* slots_d, const int32_t* s_a, int64_t n_a,
                                    int64_t a_row0, int64_t a_lo, int64_t a_hi, const int32_t* s_b,
                                    int64_t n_b, int64_t b_row0, int diag, int64_t n_f, double gamma,
                                    int rank, int world, int64_t t_lo, int64_t t_hi,
                                    uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                                    uint64_t* checksum_d, void* stream);
/* Peer-shareable device buffers for the slots (one process per GPU): cudaMalloc'd here
 * (a CUDA IPC handle must name a whole allocation; these are the only buffers the
 * library allocates, and only on request), exported as a CCC_IPC_HANDLE_BYTES handle,
 * opened in a peer process (peer access enabled lazily), closed / freed by the caller. */
ccc_status ccc_ipc_malloc(size_t bytes, void** dptr);
ccc_status ccc_ipc_free(void* dptr);
ccc_status ccc_ipc_get_handle(void* dptr, void* handle);
ccc_status ccc_ipc_open(const void* handle, void** dptr);
ccc_status ccc_ipc_close(void* dptr);

/* One block of the block-circulant 2-way decomposition (§4; §8(e)):
 * rows [a_lo, a_hi) of block A (expanded N_a / s_a / w_a, n_a rows, global index of
 * its row 0 = a_row0) against all n_b rows of block B (global row0 b_row0).
 *  diag != 0: A and B are the same block (pass the same pointers); only local pairs
 *             i<j are produced, record index = ccc_pair_index(n_b, i, j) - offset
 *             where offset = ccc_pair_index-origin of row a_lo (records of rows
 *             < a_lo are skipped, so row a_lo starts at record 0);
 *  diag == 0: every (i,j), record index (i - a_lo) * n_b + j; the caller passes
 *             the block with the lower global indices as A so that records are
 *             canonical (i < j globally).
 * Output buffers / flags as in ccc_2way.  N_a, N_b: [rows][ccc_k_pad(n_f)], 128-B
 * aligned.  If g_d != NULL the raw int32 G_ij = sum_q n_iq n_jq of every computed
 * tile is also stored at g_d[i*ldg + j] (local indices; used by the 3-way path).
 * gamma: the constant w_a / w_b were expanded with (ccc_expand).  For the paper's
 * gamma = 2/3 (compared with ==, pass 2.0/3.0) the epilogue uses the equivalent
 * integer form w(0) = (n_f + s)/(3n_f), w(1) = (3n_f - s)/(3n_f) and does not read w
 * (fewer FP64 multiplies, same result within 2 ulp); any other gamma reads w. */
ccc_status ccc_2way_block(const int8_t* N_a, const int32_t* s_a, const double* w_a,
                          int64_t n_a, int64_t a_row0, int64_t a_lo, int64_t a_hi,
                          const int8_t* N_b, const int32_t* s_b, const double* w_b,
                          int64_t n_b, int64_t b_row0, int diag, int64_t n_f, double gamma,
                          uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                          uint64_t* checksum_d, int32_t* g_d, int64_t ldg,
                          const ccc_compact* compact, void* stream);

/* 3-way preparation (§8(a) a2, a5 prerequisites): expand packed_d into the workspace
 * and compute the pairwise G = N N^T (upper triangle) that the 3-way epilogue needs. */
ccc_status ccc_3way_prepare(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                            void* ws_d, size_t ws_bytes, void* stream);

/* One 3-way stage (§8(a) a5-a6, a8; stages P:621-626) on a workspace prepared by
 * ccc_3way_prepare: for every pivot i of the stage (ccc_stage_range) the
 * Hadamard-weighted GEMM G3 = (N_{>i} o n_i) N_{>i}^T on tcgen05, then the fused
 * epilogue
 *   T111 = G3, T110 = 2G_ij - G3, T101 = 2G_ik - G3, T011 = 2G_jk - G3,
 *   T100 = 4s_i - 2G_ij - 2G_ik + G3, T010 = 4s_j - 2G_ij - 2G_jk + G3,
 *   T001 = 4s_k - 2G_ik - 2G_jk + G3,
 *   T000 = 8n_f - 4(s_i+s_j+s_k) + 2(G_ij+G_ik+G_jk) - G3,
 *   CCC(a,b,c) = T/(8n_f) * w_i(a) w_j(b) w_k(c)                 (Eq.4-5)
 * writing record t = ccc_triple_index(n_v,i,j,k) - rec_begin of every triple of the
 * stage: tallies_d uint32 [rec_count][8], ccc_d double/float [rec_count][8],
 * checksum_d as in ccc_2way.  gamma: the value given to ccc_3way_prepare (selects the
 * integer form for gamma = 2/3 as in ccc_2way_block; n_f <= 500000). */
ccc_status ccc_3way_stage(int64_t n_v, int64_t n_f, double gamma, int64_t n_stages, int64_t stage,
                          uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                          uint64_t* checksum_d, void* ws_d, size_t ws_bytes,
                          const ccc_compact* compact, void* stream);

/* One vector block as seen by the 3-way unit call: expanded rows (ccc_expand) and the
 * global index of local row 0. */
typedef struct {
    const int8_t* N;      /* [rows][ccc_k_pad(n_f)], 128-B aligned (device) */
    const int32_t* s;     /* [rows] allele-1 sums (device)                   */
    const double* w;      /* [rows][2] frequency weights (device)            */
    int64_t rows;
    int64_t row0;         /* global index of local row 0; blocks are disjoint */
} ccc_block;

/* Records produced by ccc_3way_unit for these ranges (see its layouts); -1 if invalid. */
int64_t ccc_3way_unit_records(const ccc_block* bp, int64_t p_lo, int64_t p_hi,
                              const ccc_block* bm, int64_t m_lo, int64_t m_hi,
                              const ccc_block* bn, int64_t n_lo, int64_t n_hi);

/* One unit of the tetrahedral 3-way decomposition (§4): every
 * unique triple {p, m, n} with pivot p in [p_lo,p_hi) of block bp, m in [m_lo,m_hi) of bm
 * (GEMM rows) and n in [n_lo,n_hi) of bn (GEMM columns), where bp == bm implies m > p and
 * bm == bn implies n > m (blocks are identified by row0).  `order` (0..5) says which role
 * sits in each slot of the sorted triple (i<j<k): roles p=0, m=1, n=2, orders
 * 0:(p,m,n) 1:(p,n,m) 2:(m,p,n) 3:(m,n,p) 4:(n,p,m) 5:(n,m,p); records hold the canonical
 * (Eq.5-ordered) cells.  When bp == bm the order must place p before m, when bm == bn m
 * before n (both: order 0 only), else CCC_ERR_INVALID_ARGUMENT.  G_d: the pairwise G = N N^T by GLOBAL index, G[min*ldG + max]
 * (upper triangle, e.g. from ccc_2way_block with g_d).  Record layouts:
 *   bp==bm==bn : in-block lexicographic triple order, starting at the first pivot p_lo;
 *   bp==bm     : record = (in-block pair index of (p,m) - that of (p_lo,p_lo+1)) * |N| + n-n_lo;
 *   otherwise  : ((p-p_lo)*|M| + (m-m_lo))*|N| + (n-n_lo).
 * Outputs, flags and gamma as in ccc_3way_stage; the checksum digest uses global canonical
 * indices, so unit checksums of a decomposition add up to the single-GPU checksum. */
ccc_status ccc_3way_unit(const ccc_block* bp, int64_t p_lo, int64_t p_hi, const ccc_block* bm,
                         int64_t m_lo, int64_t m_hi, const ccc_block* bn, int64_t n_lo,
                         int64_t n_hi, int order, const int32_t* G_d, int64_t ldG, int64_t n_f,
                         double gamma, uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                         uint64_t* checksum_d, const ccc_compact* compact, void* stream);

/* ccc_3way_prepare followed by ccc_3way_stage(n_stages, stage). */
ccc_status ccc_3way(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                    uint32_t out_flags, int64_t n_stages, int64_t stage, uint32_t* tallies_d,
                    void* ccc_d, uint64_t* checksum_d, void* ws_d, size_t ws_bytes,
                    const ccc_compact* compact, void* stream);

/* End-to-end 2-way with HOST buffers (the e2e measurement of bench.py): copies
 * codes_h (uint8 [n_v][n_f], pinned for full speed) to the device, packs, runs
 * ccc_2way, and copies the selected outputs back to tallies_h / ccc_h / checksum_h
 * (host, [C(n_v,2)][4] each, pinned for full speed).  Row bands of the output are
 * copied back while the next band computes.  Device scratch: dev_ws_d of at least
 * ccc_e2e_workspace_bytes(n_v, n_f, out_flags) bytes.  Synchronises `stream`
 * before returning. */
size_t ccc_e2e_workspace_bytes(int64_t n_v, int64_t n_f, uint32_t out_flags);
ccc_status ccc_2way_host(const uint8_t* codes_h, int64_t n_v, int64_t n_f, double gamma,
                         uint32_t out_flags, uint32_t* tallies_h, void* ccc_h,
                         uint64_t* checksum_h, void* dev_ws_d, size_t dev_ws_bytes,
                         void* stream);

/* 3-way end to end with stage streaming to host (SURVEY §8(f) f2 "stage streaming"; stages
 * P:621-626): H2D of codes_h (uint8 [n_v][n_f]), pack, ccc_3way_prepare, then the n_stages
 * stages of ccc_3way_stage computed into two device stage buffers in turn while a copy
 * stream drains the previous stage's records to tallies_h / ccc_h (host memory of the full
 * C(n_v,3) records, lexicographic -- pinned for overlap); checksum_h gets the whole result's
 * checksum.  dev_ws_d >= ccc_3way_host_workspace_bytes(n_v, n_f, n_stages, out_flags).
 * Returns after the last copy (synchronises `stream` and the internal copy stream). */
size_t     ccc_3way_host_workspace_bytes(int64_t n_v, int64_t n_f, int64_t n_stages, uint32_t out_flags);
ccc_status ccc_3way_host(const uint8_t* codes_h, int64_t n_v, int64_t n_f, double gamma, uint32_t out_flags,
                         int64_t n_stages, uint32_t* tallies_h, void* ccc_h, uint64_t* checksum_h,
                         void* dev_ws_d, size_t dev_ws_bytes, void* stream);

/* Number of kernels the last successful call on this thread enqueued (for the
 * bench's gpu_launches count). */
int64_t ccc_last_launch_count(void);

/* ---------------------------------------------------------------------------------
 * Sparse (missing-data) mode (§7 item 1: "the
 * value (1,0) can be set aside as a marker to denote a missing entry ... skipping
 * calculations for missing entries").  Reading A-17:
 *   present_{iq} = [code != 2],  c_i = #present,  S_i(a) over present entries,
 *   f_i(a) = S_i(a) / (2 c_i)  (0 if c_i = 0),  w_i(a) = 1 - gamma f_i(a)
 *   T_ij(a,b) over the fields where both entries are present, c_ij = their number,
 *   CCC_ij(a,b) = T_ij(a,b) / (4 c_ij) * w_i(a) * w_j(b)   (0 if c_ij = 0).
 * Records as in dense mode (lexicographic i<j, cells a-major, sum T = 4 c_ij).  On the
 * tensor pipe each pair costs four int8 MACs per field instead of one: with n = rho(1)
 * (0 if missing) and v = present, rho(0) = 2v - n, so T needs n.n, n.v, v.n and v.v.
 * --------------------------------------------------------------------------------- */

/* Rows of the sparse operand X for n_v vectors: 2 * ceil(n_v / 16) * 16. */
int64_t ccc_sparse_rows(int64_t n_v);

/* Workspace of ccc_2way_sparse (X, s, c, w); 0 if invalid. */
size_t ccc_sparse_workspace_bytes(int64_t n_v, int64_t n_f);

/* Sparse KB-expand: packed_d (ccc_pack layout) -> X_d int8 [ccc_sparse_rows(n_v)][K_pad],
 * 128-B aligned, group-interleaved: for the group g of vectors 16g..16g+15, rows
 * 32g + r hold n_{16g+r,q} (rho(1) on present entries, 0 if missing) and rows 32g + 16 + r
 * hold present_{16g+r,q} (0 on the K padding and on padding vectors >= n_v);
 * s_d int32 [n_v] = S_i(1), c_d int32 [n_v] = c_i, w_d double [n_v][2] = w_i(0), w_i(1). */
ccc_status ccc_expand_sparse(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                             int8_t* X_d, int32_t* s_d, int32_t* c_d, double* w_d, void* stream);

/* Sparse 2-way block (rows [a_lo, a_hi) of block A x all n_b vectors of block B), the
 * same record layouts, diag semantics, flags, checksum and compaction as ccc_2way_block;
 * X_a / X_b and w_a / w_b from ccc_expand_sparse of each block. */
ccc_status ccc_2way_sparse_block(const int8_t* X_a, const double* w_a, int64_t n_a, int64_t a_row0,
                                 int64_t a_lo, int64_t a_hi, const int8_t* X_b, const double* w_b,
                                 int64_t n_b, int64_t b_row0, int diag, int64_t n_f,
                                 uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                                 uint64_t* checksum_d, const ccc_compact* compact, void* stream);

/* Whole sparse 2-way problem: ccc_expand_sparse into ws_d (>= ccc_sparse_workspace_bytes,
 * 256-B aligned) then ccc_2way_sparse_block over the upper triangle; outputs as ccc_2way. */
ccc_status ccc_2way_sparse(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                           uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                           uint64_t* checksum_d, void* ws_d, size_t ws_bytes,
                           const ccc_compact* compact, void* stream);

/* ---- Sparse (missing-data) mode, 3-way (reading A-17 for triples,
 * SPEC S:303-304): T_ijk(a,b,c) over the fields where all three entries are present,
 * c_ijk = that number, f_ijk = T/(8 c_ijk), per-vector f_i(a) = S_i(a)/(2 c_i) over the
 * vector's present entries, CCC = f_ijk (1-g f_i(a))(1-g f_j(b))(1-g f_k(c)), 0 if
 * c_ijk = 0.  With n = allele-1 count (0 where missing) and v = [present],
 * rho(1) = n and rho(0) = 2v - n, so every cell is a signed sum of the 8 trilinear forms
 * sum_q x_i x_j x_k (x in {n, v}).  All 8 come out of ONE tcgen05 GEMM per (pivot, 64 j's,
 * 128 k's): B = the group-interleaved X rows (n and v) of the k's, A = the X rows of the
 * j's weighted by the pivot's n_i and by its v_i, stacked -- 8 int8 MACs per comparison,
 * no form leaves the chip (kernel tally3s.cu).
 * prepare: packed_d -> ws_d (>= ccc_sparse3_workspace_bytes): X [ccc_sparse_rows(n_v)]
 *          [K_pad] int8 (ccc_expand_sparse's layout), s_i, c_i int32, w_i(a) double
 *          (sparse weights, gamma given here).
 * stage:   records of stage `stage` of n_stages (ccc_stage_range), outputs as
 *          ccc_3way_stage (a-major cells, lexicographic triples minus the stage's first
 *          record).  ccc_3way_sparse_scratch_bytes returns 0: scratch_d / scratch_bytes
 *          are unused (kept for ABI stability; NULL is fine). */
size_t     ccc_sparse3_workspace_bytes(int64_t n_v, int64_t n_f);
size_t     ccc_3way_sparse_scratch_bytes(int64_t n_v, int64_t n_stages, int64_t stage);
ccc_status ccc_3way_sparse_prepare(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                                   void* ws_d, size_t ws_bytes, void* stream);
ccc_status ccc_3way_sparse_stage(int64_t n_v, int64_t n_f, double gamma, int64_t n_stages, int64_t stage,
                                 uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                                 void* ws_d, size_t ws_bytes, void* scratch_d, size_t scratch_bytes,
                                 void* stream);

/* ---- The paper's 3-way route on the tensor pipe, as a comparison baseline (SURVEY §8(f)
 * f4(ii); §3.2: Table 1 masks P:457-516, masked tallies P:518-525, the eight
 * reconstruction equations P:527-560 under readings A-1..A-3), with the pivot on the
 * first index: per class xi of the pivot's genotype ((0,0), heterozygote, (1,1)) one
 * masked pivot GEMM F_xi = sum_{q in xi(i)} n_jq n_kq (the paper's three mGEMM3 per
 * pivot), masked marginals Mx_xi(i,x) = sum_{q in xi(i)} n_xq (three 2-way GEMMs of the
 * masks against N, in prepare) and the class counts; then
 *   T(0,b,c) = 2 B_1(b,c) + B_2(b,c),  T(1,b,c) = 2 B_3(b,c) + B_2(b,c),
 * B_xi(1,1) = F_xi, B_xi(1,0) = 2Mx_xi(i,j) - F_xi, B_xi(0,1) = 2Mx_xi(i,k) - F_xi,
 * B_xi(0,0) = 4|xi(i)| - 2Mx_xi(i,j) - 2Mx_xi(i,k) + F_xi; CCC by Eq.4 (general gamma).
 * Same records as ccc_3way_stage (bit-identical tallies).  ws_d >= ccc_3way_paper_
 * workspace_bytes (N, s, w, 3 masks, counts, 3 n_v^2 int32 marginals); scratch_d >=
 * ccc_3way_paper_scratch_bytes (2 stored forms per record).  Not the product path. */
size_t     ccc_3way_paper_workspace_bytes(int64_t n_v, int64_t n_f);
size_t     ccc_3way_paper_scratch_bytes(int64_t n_v, int64_t n_stages, int64_t stage);
ccc_status ccc_3way_paper_prepare(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma, void* ws_d,
                                  size_t ws_bytes, void* stream);
ccc_status ccc_3way_paper_stage(int64_t n_v, int64_t n_f, double gamma, int64_t n_stages, int64_t stage,
                                uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                                void* ws_d, size_t ws_bytes, void* scratch_d, size_t scratch_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CCC_H_ */
