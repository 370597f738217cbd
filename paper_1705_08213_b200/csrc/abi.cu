// abi.cu -- the extern "C" boundary of libccc (include/ccc.h): argument validation,
// workspace layout, TMA descriptor construction and kernel launches.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "ccc.h"
#include "internal.h"

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;

ccc_status fail(ccc_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

ccc_status cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return CCC_ERR_CUDA;
}

#define CCC_CUDA(call, what)                              \
    do {                                                  \
        cudaError_t e_ = (call);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

#define CCC_CHECK(call)                      \
    do {                                     \
        ccc_status st_ = (call);             \
        if (st_ != CCC_OK) return st_;       \
    } while (0)

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int64_t c2(int64_t n) { return n < 2 ? 0 : n * (n - 1) / 2; }
int64_t c3(int64_t n) { return n < 3 ? 0 : n * (n - 1) * (n - 2) / 6; }
int64_t kpad_of(int64_t n_f) { return (n_f + 127) / 128 * 128; }
int64_t pstride_of(int64_t n_f) { return (n_f + 63) / 64 * 16; }

struct DevInfo {
    int sms = 0, major = 0, minor = 0;
    bool valid = false;
};
std::mutex g_dev_mu;
DevInfo g_dev[64];

ccc_status check_device(int* num_sms) {
    int dev = 0;
    CCC_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= 64) return fail(CCC_ERR_UNSUPPORTED, "device ordinal out of range");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevInfo& d = g_dev[dev];
    if (!d.valid) {
        CCC_CUDA(cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev),
                 "cudaDeviceGetAttribute");
        CCC_CUDA(cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev),
                 "cudaDeviceGetAttribute");
        CCC_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev),
                 "cudaDeviceGetAttribute");
        d.valid = true;
    }
    if (d.major != 10 || d.minor != 0) {
        char buf[128];
        snprintf(buf, sizeof buf, "device is sm_%d%d; libccc is built for sm_100a only", d.major,
                 d.minor);
        return fail(CCC_ERR_UNSUPPORTED, buf);
    }
    *num_sms = d.sms;
    return CCC_OK;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

ccc_status get_encode(EncodeTiledFn* out) {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        if (err == cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) return fail(CCC_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    *out = fn;
    return CCC_OK;
}

// 2-D uint8 tensor map over an expanded N block [rows][k_pad], box = 128 B x box_rows,
// 128-byte swizzle (matches the UMMA SWIZZLE_128B K-major smem descriptor).
ccc_status make_tmap(CUtensorMap* tm, const void* base, int64_t rows, int64_t k_pad,
                     uint32_t box_rows) {
    EncodeTiledFn enc;
    CCC_CHECK(get_encode(&enc));
    cuuint64_t dims[2] = {(cuuint64_t)k_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)k_pad};
    cuuint32_t box[2] = {(cuuint32_t)ccc::kBK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[96];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
        return fail(CCC_ERR_CUDA, buf);
    }
    return CCC_OK;
}

ccc_status check_sizes(int64_t n_v, int64_t n_f) {
    if (n_v < 0) return fail(CCC_ERR_INVALID_ARGUMENT, "n_v must be >= 0");
    if (n_f < 1) return fail(CCC_ERR_INVALID_ARGUMENT, "n_f must be >= 1");
    if (n_f > CCC_MAX_NF) return fail(CCC_ERR_UNSUPPORTED, "n_f exceeds CCC_MAX_NF (8 n_f must fit int32)");
    if (n_v > CCC_MAX_NV) return fail(CCC_ERR_UNSUPPORTED, "n_v exceeds CCC_MAX_NV");
    return CCC_OK;
}

ccc_status check_compact(const ccc_compact* c) {
    if (!c) return CCC_OK;
    if (c->capacity < 0) return fail(CCC_ERR_INVALID_ARGUMENT, "compact capacity must be >= 0");
    if (!c->count_d || !aligned(c->count_d, 8))
        return fail(CCC_ERR_INVALID_ARGUMENT, "compact count_d must be a non-NULL 8-B aligned pointer");
    if (c->capacity > 0 && (!c->keys_d || !aligned(c->keys_d, 8)))
        return fail(CCC_ERR_INVALID_ARGUMENT, "compact keys_d must be a non-NULL 8-B aligned pointer");
    if (c->threshold != c->threshold) return fail(CCC_ERR_INVALID_ARGUMENT, "compact threshold is NaN");
    return CCC_OK;
}

ccc::Compact to_compact(const ccc_compact* c) {
    ccc::Compact k{};
    if (c) {
        k.thr = c->threshold;
        k.cap = c->capacity;
        k.keys = reinterpret_cast<unsigned long long*>(c->keys_d);
        k.count = reinterpret_cast<unsigned long long*>(c->count_d);
    }
    return k;
}

ccc_status check_outputs(uint32_t flags, const uint32_t* tallies, const void* ccc,
                         const uint64_t* ck) {
    if (flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if ((flags & CCC_OUT_CCC_F64) && (flags & CCC_OUT_CCC_F32))
        return fail(CCC_ERR_INVALID_ARGUMENT, "CCC_OUT_CCC_F64 and CCC_OUT_CCC_F32 are exclusive");
    if ((flags & CCC_OUT_TALLY) && (!tallies || !aligned(tallies, 16)))
        return fail(CCC_ERR_INVALID_ARGUMENT, "tallies must be a non-NULL 16-B aligned pointer");
    if ((flags & (CCC_OUT_CCC_F64 | CCC_OUT_CCC_F32)) && (!ccc || !aligned(ccc, 16)))
        return fail(CCC_ERR_INVALID_ARGUMENT, "ccc must be a non-NULL 16-B aligned pointer");
    if ((flags & CCC_OUT_CHECKSUM) && (!ck || !aligned(ck, 8)))
        return fail(CCC_ERR_INVALID_ARGUMENT, "checksum must be a non-NULL 8-B aligned pointer");
    return CCC_OK;
}

// B operand of the 3-way pivot GEMM as the 4-D view (K, a: 2 [stride 4 rows], b: 4 [1 row],
// g [8 rows]) of a row-major [rows][k_pad] matrix: a 128-row box lands in shared memory as
// row 8g + 2b + a <- n = 8g + 4a + b (tally3_kernel's args.permb).  Needs the memory of
// ceil8(rows) rows to be readable: `readable_rows` says how many the buffer holds; with
// fewer the plain 2-D map is made and *permb = 0 (rows past `rows` are masked columns).
ccc_status make_tmap_b3(CUtensorMap* tm, const void* base, int64_t rows, int64_t readable_rows, int64_t k_pad,
                        int32_t* permb) {
    const int64_t r8 = (rows + 7) / 8 * 8;
    if (readable_rows < r8) {
        *permb = 0;
        return make_tmap(tm, base, rows, k_pad, 128);
    }
    EncodeTiledFn enc;
    CCC_CHECK(get_encode(&enc));
    cuuint64_t dims[4] = {(cuuint64_t)k_pad, 2, 4, (cuuint64_t)(r8 / 8)};
    cuuint64_t strides[3] = {(cuuint64_t)(4 * k_pad), (cuuint64_t)k_pad, (cuuint64_t)(8 * k_pad)};
    cuuint32_t box[4] = {(cuuint32_t)ccc::kBK, 2, 4, 16};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char buf[96];
        snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled (4-D) failed (CUresult %d)", (int)r);
        return fail(CCC_ERR_CUDA, buf);
    }
    *permb = 1;
    return CCC_OK;
}


struct WsLayout {
    size_t N = 0, s = 0, w = 0, G = 0, total = 0;
};

WsLayout ws_layout(int way, int64_t n_v, int64_t n_f) {
    WsLayout L;
    size_t off = 0;
    L.N = off;   // rows padded to a multiple of 8: the 3-way B operand's 4-D view reads them
    off += al256((size_t)((n_v + 7) / 8 * 8) * (size_t)kpad_of(n_f));
    L.s = off;
    off += al256((size_t)n_v * 4);
    L.w = off;
    off += al256((size_t)n_v * 16);
    if (way == 3) {
        L.G = off;
        off += al256((size_t)n_v * (size_t)n_v * 4);
    }
    L.total = off + 256;  // slack so a caller base need only be 256-B aligned
    return L;
}

// gamma == 2/3 exactly as the caller computed it (2.0/3.0 in C, 2/3 in Python): the
// weights are then w(a) = U(a) / (3 n_f) with integer U, and the epilogues form CCC
// from integer products instead of the stored doubles (K-2).
bool is_gamma23(double gamma) { return gamma == 2.0 / 3.0; }

// 3-way: CCC = (T U_p U_m) U_n / (216 n_f^4); T U_p U_m <= 72 n_f^3 stays below 2^63
// (and exact in double below 2^53, n_f <= 50000) for n_f <= 500000.
void set_exact3(ccc::Tally3Args& a, int64_t n_f, double gamma) {
    a.exact23 = (is_gamma23(gamma) && n_f <= 500000) ? 1 : 0;
    // T U_p U_m <= 8 n_f (3 n_f)^2 = 72 n_f^3 < 2^52 (n_f <= 38,000): the FULL epilogue
    // builds 2^52 + T U_p U_m as a double's bit pattern and needs one DFMA per cell
    a.exact52 = (a.exact23 && 72.0 * (double)n_f * (double)n_f * (double)n_f < 4503599627370496.0) ? 1 : 0;
    const double nf = (double)n_f;
    a.inv_d = 1.0 / (216.0 * nf * nf * nf * nf);
}

ccc_status block_impl(const int8_t* N_a, const int32_t* s_a, const double* w_a, int64_t n_a,
                      int64_t a_row0, int64_t a_lo, int64_t a_hi, const int8_t* N_b,
                      const int32_t* s_b, const double* w_b, int64_t n_b, int64_t b_row0,
                      int diag, int64_t n_f, double gamma, uint32_t flags, uint32_t* tallies,
                      void* ccc, uint64_t* ck, int32_t* g, int64_t ldg,
                      const ccc_compact* cmp, cudaStream_t stream, int num_sms) {
    const int64_t k_pad = kpad_of(n_f);
    CUtensorMap tmA, tmB;
    CCC_CHECK(make_tmap(&tmA, N_a, n_a, k_pad, ccc::kBM));
    CCC_CHECK(make_tmap(&tmB, N_b, n_b, k_pad, (uint32_t)ccc::tally2_b_box_rows()));
    ccc::Tally2Args a{};
    a.a_lo = a_lo;
    a.nA = a_hi - a_lo;
    a.nB = n_b;
    a.a_row0 = a_row0;
    a.b_row0 = b_row0;
    a.diag = diag ? 1 : 0;
    a.n_f = (int32_t)n_f;
    a.k_blocks = (int32_t)(k_pad / ccc::kBK);
    a.out_flags = (int32_t)flags;
    // gamma = 2/3: CCC = (T U_i(a)) U_j(b) / (36 n_f^3) from integers (K-2)
    a.exact23 = is_gamma23(gamma) ? 1 : 0;
    a.inv_d = 1.0 / (36.0 * (double)n_f * (double)n_f * (double)n_f);
    a.compact = cmp ? 1 : 0;
    a.cmp = to_compact(cmp);
    a.s_a = s_a;
    a.s_b = s_b;
    a.w_a = w_a;
    a.w_b = w_b;
    a.tallies = tallies;
    a.ccc = ccc;
    a.checksum = reinterpret_cast<unsigned long long*>(ck);
    a.g_out = g;
    a.ldg = ldg;
    a.rec_row_base = diag ? (a_lo * (2 * n_b - a_lo - 1)) / 2 : 0;
    a.sup_rows = 2048;
    a.sup_cols = 2048;   // 2048 x 2048-element super tiles (measured best)
    int64_t tiles = 0;
    CCC_CUDA(ccc::launch_tally2(tmA, tmB, a, num_sms, stream, &tiles), "tally2 launch");
    if (tiles) ++g_launches;
    return CCC_OK;
}

}  // namespace

extern "C" {

int ccc_version(void) { return 100; }

const char* ccc_status_string(int st) {
    switch (st) {
        case CCC_OK: return "CCC_OK";
        case CCC_ERR_INVALID_ARGUMENT: return "CCC_ERR_INVALID_ARGUMENT";
        case CCC_ERR_UNSUPPORTED: return "CCC_ERR_UNSUPPORTED";
        case CCC_ERR_CUDA: return "CCC_ERR_CUDA";
        case CCC_ERR_WORKSPACE: return "CCC_ERR_WORKSPACE";
        default: return "CCC_ERR_UNKNOWN";
    }
}

const char* ccc_last_error(void) { return g_err.c_str(); }

int64_t ccc_last_launch_count(void) { return g_launches; }

int64_t ccc_num_unique(int num_way, int64_t n_v) {
    if (num_way == 2) return c2(n_v);
    if (num_way == 3) return c3(n_v);
    return -1;
}

int64_t ccc_pair_index(int64_t n_v, int64_t i, int64_t j) {
    if (!(0 <= i && i < j && j < n_v)) return -1;
    return i * (2 * n_v - i - 1) / 2 + (j - i - 1);
}

int64_t ccc_triple_index(int64_t n_v, int64_t i, int64_t j, int64_t k) {
    if (!(0 <= i && i < j && j < k && k < n_v)) return -1;
    return c3(n_v) - c3(n_v - i) + c2(n_v - i - 1) - c2(n_v - j) + (k - j - 1);
}

int64_t ccc_packed_stride(int64_t n_f) { return n_f < 1 ? -1 : pstride_of(n_f); }

int64_t ccc_k_pad(int64_t n_f) { return n_f < 1 ? -1 : kpad_of(n_f); }

ccc_status ccc_stage_range(int64_t n_v, int64_t n_stages, int64_t stage, int64_t* out) {
    if (!out) return fail(CCC_ERR_INVALID_ARGUMENT, "out must not be NULL");
    if (n_v < 0 || n_stages < 1 || stage < 0 || stage >= n_stages)
        return fail(CCC_ERR_INVALID_ARGUMENT, "need n_v >= 0, n_stages >= 1, 0 <= stage < n_stages");
    const int64_t tot = c3(n_v);
    // cum(i) = records of pivots < i = C(n_v,3) - C(n_v-i,3); stage boundary b(s) is the
    // smallest i with cum(i) >= ceil(s * tot / n_stages).
    auto cum = [&](int64_t i) { return tot - c3(n_v - i); };
    auto bound = [&](int64_t s) -> int64_t {
        if (s <= 0) return 0;
        if (s >= n_stages) return n_v;
        const __int128 t = (__int128)s * tot;
        const int64_t target = (int64_t)((t + n_stages - 1) / n_stages);
        int64_t lo = 0, hi = n_v;  // cum(n_v) = tot >= target
        while (lo < hi) {
            int64_t mid = (lo + hi) / 2;
            if (cum(mid) >= target) hi = mid;
            else lo = mid + 1;
        }
        return lo;
    };
    const int64_t ib = bound(stage), ie = bound(stage + 1);
    out[0] = ib;
    out[1] = ie;
    out[2] = cum(ib);
    out[3] = cum(ie) - cum(ib);
    return CCC_OK;
}

size_t ccc_workspace_bytes(int num_way, int64_t n_v, int64_t n_f) {
    if ((num_way != 2 && num_way != 3) || n_v < 0 || n_f < 1) return 0;
    return ws_layout(num_way, n_v, n_f).total;
}

ccc_status ccc_pack(const uint8_t* codes_d, int64_t n_v, int64_t n_f, uint8_t* packed_d,
                    void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v == 0) return CCC_OK;
    if (!codes_d || !packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "codes_d / packed_d must be non-NULL, packed_d 16-B aligned");
    int sms;
    CCC_CHECK(check_device(&sms));
    CCC_CUDA(ccc::launch_pack(codes_d, n_v, n_f, packed_d, sms, (cudaStream_t)stream), "pack launch");
    g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_expand(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                      int8_t* N_d, int32_t* s_d, double* w_d, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v == 0) return CCC_OK;
    if (!packed_d || !N_d || !s_d || !w_d || !aligned(packed_d, 16) || !aligned(N_d, 128) ||
        !aligned(s_d, 4) || !aligned(w_d, 8))
        return fail(CCC_ERR_INVALID_ARGUMENT,
                    "packed_d (16-B), N_d (128-B), s_d, w_d must be non-NULL and aligned");
    int sms;
    CCC_CHECK(check_device(&sms));
    CCC_CUDA(ccc::launch_expand(packed_d, n_v, n_f, gamma, N_d, s_d, w_d, sms, (cudaStream_t)stream),
             "expand launch");
    g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_expand_codes(const uint8_t* codes_d, int64_t n_v, int64_t n_f, double gamma,
                            int8_t* N_d, int32_t* s_d, double* w_d, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v == 0) return CCC_OK;
    if (!codes_d || !N_d || !s_d || !w_d || !aligned(N_d, 128) || !aligned(s_d, 4) || !aligned(w_d, 8))
        return fail(CCC_ERR_INVALID_ARGUMENT, "codes_d, N_d (128-B), s_d, w_d must be non-NULL and aligned");
    int sms;
    CCC_CHECK(check_device(&sms));
    CCC_CUDA(ccc::launch_expand_codes(codes_d, n_v, n_f, gamma, N_d, s_d, w_d, sms, (cudaStream_t)stream),
             "expand_codes launch");
    g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_2way_block(const int8_t* N_a, const int32_t* s_a, const double* w_a, int64_t n_a,
                          int64_t a_row0, int64_t a_lo, int64_t a_hi, const int8_t* N_b,
                          const int32_t* s_b, const double* w_b, int64_t n_b, int64_t b_row0,
                          int diag, int64_t n_f, double gamma, uint32_t out_flags, uint32_t* tallies_d,
                          void* ccc_d, uint64_t* checksum_d, int32_t* g_d, int64_t ldg,
                          const ccc_compact* compact, void* stream) {
    CCC_CHECK(check_compact(compact));
    g_launches = 0;
    CCC_CHECK(check_sizes(n_a, n_f));
    CCC_CHECK(check_sizes(n_b, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (!(0 <= a_lo && a_lo <= a_hi && a_hi <= n_a))
        return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= a_lo <= a_hi <= n_a");
    if (diag && (N_a != N_b || n_a != n_b || a_row0 != b_row0))
        return fail(CCC_ERR_INVALID_ARGUMENT, "diag block needs A == B");
    if (a_row0 < 0 || b_row0 < 0 || a_row0 + n_a > CCC_MAX_NV || b_row0 + n_b > CCC_MAX_NV)
        return fail(CCC_ERR_INVALID_ARGUMENT, "global row indices out of range");
    if (g_d && ldg < n_b) return fail(CCC_ERR_INVALID_ARGUMENT, "ldg must be >= n_b");
    if (a_hi == a_lo || n_b == 0) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!N_a || !N_b || !s_a || !s_b || !w_a || !w_b || !aligned(N_a, 128) || !aligned(N_b, 128))
        return fail(CCC_ERR_INVALID_ARGUMENT, "N_a/N_b (128-B aligned), s, w must be non-NULL");
    int sms;
    CCC_CHECK(check_device(&sms));
    return block_impl(N_a, s_a, w_a, n_a, a_row0, a_lo, a_hi, N_b, s_b, w_b, n_b, b_row0, diag,
                      n_f, gamma, out_flags, tallies_d, ccc_d, checksum_d, g_d, ldg, compact,
                      (cudaStream_t)stream, sms);
}

ccc_status ccc_2way(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                    uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                    void* ws_d, size_t ws_bytes, const ccc_compact* compact, void* stream) {
    CCC_CHECK(check_compact(compact));
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (n_v < 2) return CCC_OK;  // empty result: nothing to write
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "packed_d must be non-NULL and 16-B aligned");
    const WsLayout L = ws_layout(2, n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    int8_t* N = reinterpret_cast<int8_t*>(ws + L.N);
    int32_t* s = reinterpret_cast<int32_t*>(ws + L.s);
    double* w = reinterpret_cast<double*>(ws + L.w);
    cudaStream_t st = (cudaStream_t)stream;
    CCC_CUDA(ccc::launch_expand(packed_d, n_v, n_f, gamma, N, s, w, sms, st), "expand launch");
    CCC_CHECK(block_impl(N, s, w, n_v, 0, 0, n_v, N, s, w, n_v, 0, 1, n_f, gamma, out_flags, tallies_d,
                         ccc_d, checksum_d, nullptr, 0, compact, st, sms));
    g_launches += 1;
    return CCC_OK;
}

ccc_status ccc_2way_codes(const uint8_t* codes_d, int64_t n_v, int64_t n_f, double gamma, uint32_t out_flags,
                          uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d, void* ws_d, size_t ws_bytes,
                          const ccc_compact* compact, void* stream) {
    CCC_CHECK(check_compact(compact));
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (n_v < 2) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!codes_d) return fail(CCC_ERR_INVALID_ARGUMENT, "codes_d must be non-NULL");
    const WsLayout L = ws_layout(2, n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    int8_t* N = reinterpret_cast<int8_t*>(ws + L.N);
    int32_t* s = reinterpret_cast<int32_t*>(ws + L.s);
    double* w = reinterpret_cast<double*>(ws + L.w);
    cudaStream_t st = (cudaStream_t)stream;
    // unpacked codes straight to the operand (no 2-bit intermediate on one GPU), then the
    // fused tally GEMM; running the expand concurrently with the GEMM (producer waiting per
    // 128-row block) was measured slower (profiles/r02_experiments.md)
    CCC_CUDA(ccc::launch_expand_codes(codes_d, n_v, n_f, gamma, N, s, w, sms, st), "expand_codes launch");
    CCC_CHECK(block_impl(N, s, w, n_v, 0, 0, n_v, N, s, w, n_v, 0, 1, n_f, gamma, out_flags, tallies_d, ccc_d,
                         checksum_d, nullptr, 0, compact, st, sms));
    g_launches += 1;
    return CCC_OK;
}

ccc_status ccc_2way_popcount(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                             uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                             uint64_t* checksum_d, void* ws_d, size_t ws_bytes, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (n_v < 2) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "packed_d must be non-NULL and 16-B aligned");
    const WsLayout L = ws_layout(2, n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    CCC_CUDA(ccc::launch_popc_2way(packed_d, n_v, n_f, gamma, out_flags, tallies_d, ccc_d,
                                   reinterpret_cast<unsigned long long*>(checksum_d),
                                   reinterpret_cast<int32_t*>(ws + L.s), reinterpret_cast<double*>(ws + L.w),
                                   sms, (cudaStream_t)stream),
             "popcount launch");
    g_launches = 2;
    return CCC_OK;
}

// ---------------------------------------------------------------- f3: field split
namespace {
ccc_status fs_geom(int64_t n_a, int64_t a_row0, int64_t a_lo, int64_t a_hi, int64_t n_b, int64_t b_row0,
                   int diag, ccc::FsGeom* g) {
    if (n_a < 0 || n_b < 0 || !(0 <= a_lo && a_lo <= a_hi && a_hi <= n_a))
        return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= a_lo <= a_hi <= n_a and n_b >= 0");
    if (diag && n_a != n_b) return fail(CCC_ERR_INVALID_ARGUMENT, "diag block needs n_a == n_b");
    if (a_row0 < 0 || b_row0 < 0 || a_row0 + n_a > CCC_MAX_NV || b_row0 + n_b > CCC_MAX_NV)
        return fail(CCC_ERR_INVALID_ARGUMENT, "global row indices out of range");
    *g = ccc::FsGeom{};
    g->a_lo = a_lo;
    g->nA = a_hi - a_lo;
    g->nB = n_b;
    g->a_row0 = a_row0;
    g->b_row0 = b_row0;
    g->diag = diag ? 1 : 0;
    return CCC_OK;
}

ccc_status fs_export_impl(const int8_t* N_a, const int32_t* s_a, int64_t n_a, const int8_t* N_b,
                          const int32_t* s_b, const ccc::FsGeom& g, int64_t n_f_slice, int32_t* const* slots_d,
                          int rank, int world, int64_t t_lo, int64_t t_hi, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_a, n_f_slice));
    CCC_CHECK(check_sizes(g.nB, n_f_slice));
    if (world < 1 || rank < 0 || rank >= world) return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= rank < world");
    if (t_lo < 0 || t_hi < t_lo) return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= t_lo <= t_hi");
    if (g.nA == 0 || g.nB == 0 || t_hi == t_lo) return CCC_OK;
    if (g.diag && N_a != N_b) return fail(CCC_ERR_INVALID_ARGUMENT, "diag block needs A == B");
    if (!N_a || !N_b || !aligned(N_a, 128) || !aligned(N_b, 128) || !s_a || !s_b || !slots_d)
        return fail(CCC_ERR_INVALID_ARGUMENT, "N (128-B aligned), s and slots_d must be non-NULL");
    int sms;
    CCC_CHECK(check_device(&sms));
    const int64_t k_pad = kpad_of(n_f_slice);
    CUtensorMap tmA, tmB;
    CCC_CHECK(make_tmap(&tmA, N_a, n_a, k_pad, ccc::kBM));
    CCC_CHECK(make_tmap(&tmB, N_b, g.nB, k_pad, (uint32_t)ccc::tally2_b_box_rows()));
    ccc::Tally2Args a{};
    a.a_lo = g.a_lo;
    a.nA = g.nA;
    a.nB = g.nB;
    a.a_row0 = g.a_row0;
    a.b_row0 = g.b_row0;
    a.diag = g.diag;
    a.n_f = (int32_t)n_f_slice;
    a.k_blocks = (int32_t)(k_pad / ccc::kBK);
    a.out_flags = 0;
    a.exact23 = 1;          // the per-row setup then reads s only (no w)
    a.s_a = s_a;
    a.s_b = s_b;
    a.sup_rows = a.sup_cols = 2048;   // the schedule ccc_2way_fs_finish walks
    a.t_lo = t_lo;
    a.t_hi = t_hi;
    a.xp_ptrs = slots_d;
    a.xp_rank = rank;
    a.xp_world = world;
    int64_t tiles = 0;
    CCC_CUDA(ccc::launch_tally2(tmA, tmB, a, sms, (cudaStream_t)stream, &tiles), "fs export launch");
    if (tiles) ++g_launches;
    return CCC_OK;
}

ccc_status fs_finish_impl(const int32_t* slots_d, const int32_t* s_a, const int32_t* s_b, const ccc::FsGeom& g,
                          int64_t n_f, double gamma, int rank, int world, int64_t t_lo, int64_t t_hi,
                          uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                          void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(g.nB, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (world < 1 || rank < 0 || rank >= world) return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= rank < world");
    if (t_lo < 0 || t_hi < t_lo) return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= t_lo <= t_hi");
    if (g.nA == 0 || g.nB == 0 || t_hi == t_lo) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!slots_d || !s_a || !s_b) return fail(CCC_ERR_INVALID_ARGUMENT, "slots_d and s must be non-NULL");
    int sms;
    CCC_CHECK(check_device(&sms));
    CCC_CUDA(ccc::launch_fs_finish(slots_d, s_a, s_b, g, n_f, gamma, rank, world, t_lo, t_hi, out_flags,
                                   tallies_d, ccc_d, reinterpret_cast<unsigned long long*>(checksum_d),
                                   sms, (cudaStream_t)stream),
             "fs finish launch");
    ++g_launches;
    return CCC_OK;
}
}  // namespace

int64_t ccc_2way_fs_tiles(int64_t n_v) { return n_v < 2 ? 0 : ccc::fs_total_tiles(n_v); }

int64_t ccc_2way_fs_block_tiles(int64_t n_a, int64_t a_lo, int64_t a_hi, int64_t n_b, int diag) {
    ccc::FsGeom g;
    if (fs_geom(n_a, 0, a_lo, a_hi, n_b, 0, diag, &g) != CCC_OK) return -1;
    if (g.nA == 0 || g.nB == 0) return 0;
    return ccc::fs_block_tiles(g);
}

size_t ccc_2way_fs_slot_bytes(int world, int64_t t_lo, int64_t t_hi) {
    if (world < 1 || t_hi <= t_lo) return 0;
    const int64_t owned = (t_hi - t_lo + world - 1) / world;
    return (size_t)owned * (size_t)world * 65536u * sizeof(int32_t);
}

ccc_status ccc_2way_fs_export(const int8_t* N_d, const int32_t* s_d, int64_t n_v, int64_t n_f_slice,
                              int32_t* const* slots_d, int rank, int world, int64_t t_lo, int64_t t_hi,
                              void* stream) {
    g_launches = 0;
    ccc::FsGeom g;
    CCC_CHECK(fs_geom(n_v, 0, 0, n_v, n_v, 0, 1, &g));
    if (n_v < 2) return CCC_OK;
    return fs_export_impl(N_d, s_d, n_v, N_d, s_d, g, n_f_slice, slots_d, rank, world, t_lo, t_hi, stream);
}

ccc_status ccc_2way_fs_finish(const int32_t* slots_d, const int32_t* s_d, int64_t n_v, int64_t n_f,
                              double gamma, int rank, int world, int64_t t_lo, int64_t t_hi,
                              uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                              void* stream) {
    g_launches = 0;
    ccc::FsGeom g;
    CCC_CHECK(fs_geom(n_v, 0, 0, n_v, n_v, 0, 1, &g));
    if (n_v < 2) return CCC_OK;
    return fs_finish_impl(slots_d, s_d, s_d, g, n_f, gamma, rank, world, t_lo, t_hi, out_flags, tallies_d,
                          ccc_d, checksum_d, stream);
}

ccc_status ccc_2way_fs_block_export(const int8_t* N_a, const int32_t* s_a, int64_t n_a, int64_t a_lo,
                                    int64_t a_hi, const int8_t* N_b, const int32_t* s_b, int64_t n_b, int diag,
                                    int64_t n_f_slice, int32_t* const* slots_d, int rank, int world,
                                    int64_t t_lo, int64_t t_hi, void* stream) {
    g_launches = 0;
    ccc::FsGeom g;
    CCC_CHECK(fs_geom(n_a, 0, a_lo, a_hi, n_b, 0, diag, &g));
    return fs_export_impl(N_a, s_a, n_a, N_b, s_b, g, n_f_slice, slots_d, rank, world, t_lo, t_hi, stream);
}

ccc_status ccc_2way_fs_block_finish(const int32_t* slots_d, const int32_t* s_a, int64_t n_a, int64_t a_row0,
                                    int64_t a_lo, int64_t a_hi, const int32_t* s_b, int64_t n_b, int64_t b_row0,
                                    int diag, int64_t n_f, double gamma, int rank, int world, int64_t t_lo,
                                    int64_t t_hi, uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                                    uint64_t* checksum_d, void* stream) {
    g_launches = 0;
    ccc::FsGeom g;
    CCC_CHECK(fs_geom(n_a, a_row0, a_lo, a_hi, n_b, b_row0, diag, &g));
    if (diag && s_a != s_b) return fail(CCC_ERR_INVALID_ARGUMENT, "diag block needs s_a == s_b");
    return fs_finish_impl(slots_d, s_a, s_b, g, n_f, gamma, rank, world, t_lo, t_hi, out_flags, tallies_d,
                          ccc_d, checksum_d, stream);
}

ccc_status ccc_ipc_malloc(size_t bytes, void** dptr) {
    if (!dptr || bytes == 0) return fail(CCC_ERR_INVALID_ARGUMENT, "dptr non-NULL, bytes > 0");
    CCC_CUDA(cudaMalloc(dptr, bytes), "cudaMalloc (ipc buffer)");
    return CCC_OK;
}

ccc_status ccc_ipc_free(void* dptr) {
    CCC_CUDA(cudaFree(dptr), "cudaFree (ipc buffer)");
    return CCC_OK;
}

ccc_status ccc_ipc_get_handle(void* dptr, void* handle) {
    if (!dptr || !handle) return fail(CCC_ERR_INVALID_ARGUMENT, "dptr and handle must be non-NULL");
    static_assert(sizeof(cudaIpcMemHandle_t) == CCC_IPC_HANDLE_BYTES, "ipc handle size");
    CCC_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), dptr), "cudaIpcGetMemHandle");
    return CCC_OK;
}

ccc_status ccc_ipc_open(const void* handle, void** dptr) {
    if (!dptr || !handle) return fail(CCC_ERR_INVALID_ARGUMENT, "dptr and handle must be non-NULL");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    CCC_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return CCC_OK;
}

ccc_status ccc_ipc_close(void* dptr) {
    CCC_CUDA(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
    return CCC_OK;
}

ccc_status ccc_3way_prepare(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                            void* ws_d, size_t ws_bytes, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v < 3) return CCC_OK;
    if (!packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "packed_d must be non-NULL and 16-B aligned");
    const WsLayout L = ws_layout(3, n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    int8_t* N = reinterpret_cast<int8_t*>(ws + L.N);
    int32_t* s = reinterpret_cast<int32_t*>(ws + L.s);
    double* w = reinterpret_cast<double*>(ws + L.w);
    int32_t* G = reinterpret_cast<int32_t*>(ws + L.G);
    cudaStream_t st = (cudaStream_t)stream;
    CCC_CUDA(ccc::launch_expand(packed_d, n_v, n_f, gamma, N, s, w, sms, st), "expand launch");
    CCC_CHECK(block_impl(N, s, w, n_v, 0, 0, n_v, N, s, w, n_v, 0, 1, n_f, gamma, 0, nullptr, nullptr,
                         nullptr, G, n_v, nullptr, st, sms));
    g_launches += 1;
    return CCC_OK;
}

ccc_status ccc_3way_stage(int64_t n_v, int64_t n_f, double gamma, int64_t n_stages, int64_t stage,
                          uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                          uint64_t* checksum_d, void* ws_d, size_t ws_bytes, const ccc_compact* compact, void* stream) {
    CCC_CHECK(check_compact(compact));
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    int64_t rng[4];
    CCC_CHECK(ccc_stage_range(n_v, n_stages, stage, rng));
    if (n_v < 3 || rng[3] == 0) return CCC_OK;  // empty stage: nothing to write
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    const WsLayout L = ws_layout(3, n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    const int64_t k_pad = kpad_of(n_f);
    ccc::Blk3 b{reinterpret_cast<const int8_t*>(ws + L.N), reinterpret_cast<const int32_t*>(ws + L.s),
                reinterpret_cast<const double*>(ws + L.w), n_v, 0};
    ccc::Tally3Args a{};
    a.bp = a.bm = a.bn = b;
    a.p_lo = rng[0];
    a.p_hi = rng[1];
    a.m_lo = 0;
    a.m_hi = n_v;
    a.n_lo = 0;
    a.n_hi = n_v;
    a.same_pm = a.same_mn = 1;
    a.order = 0;
    a.layout = 0;
    a.ppair = 1;
    a.G = reinterpret_cast<const int32_t*>(ws + L.G);
    a.ldG = n_v;
    a.rec_base = rng[2];
    a.k_pad = k_pad;
    a.n_f = (int32_t)n_f;
    a.k_blocks = (int32_t)(k_pad / ccc::kBK);
    a.out_flags = (int32_t)out_flags;
    set_exact3(a, n_f, gamma);
    a.compact = compact ? 1 : 0;
    a.cmp = to_compact(compact);
    a.tallies = tallies_d;
    a.ccc = ccc_d;
    a.checksum = reinterpret_cast<unsigned long long*>(checksum_d);
    CUtensorMap tmA, tmB;
    CCC_CHECK(make_tmap(&tmA, b.N, n_v, k_pad, 128));
    CCC_CHECK(make_tmap_b3(&tmB, b.N, n_v, (n_v + 7) / 8 * 8, k_pad, &a.permb));   // workspace: padded
    int64_t units = 0;
    CCC_CUDA(ccc::launch_tally3(tmA, tmB, a, sms, (cudaStream_t)stream, &units), "tally3 launch");
    if (units) g_launches = 1;
    return CCC_OK;
}

// ---------------------------------------------------------------- f1: sparse 3-way
namespace {
// workspace: the group-interleaved X of the sparse mode (ccc_expand_sparse's layout), s, c, w
struct Sp3Layout {
    size_t X = 0, s = 0, c = 0, w = 0, total = 0;
};
Sp3Layout sp3_layout(int64_t n_v, int64_t n_f) {
    Sp3Layout L;
    size_t off = 0;
    L.X = off;
    off += al256((size_t)(2 * ((n_v + 15) / 16 * 16)) * (size_t)kpad_of(n_f));
    L.s = off;
    off += al256((size_t)n_v * 4);
    L.c = off;
    off += al256((size_t)n_v * 4);
    L.w = off;
    off += al256((size_t)n_v * 16);
    L.total = off + 256;
    return L;
}
}  // namespace

size_t ccc_sparse3_workspace_bytes(int64_t n_v, int64_t n_f) {
    if (n_v < 0 || n_f < 1) return 0;
    return sp3_layout(n_v, n_f).total;
}

size_t ccc_3way_sparse_scratch_bytes(int64_t n_v, int64_t n_stages, int64_t stage) {
    (void)n_v;
    (void)n_stages;
    (void)stage;
    return 0;   // single pass: no stored forms
}

ccc_status ccc_3way_sparse_prepare(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                                   void* ws_d, size_t ws_bytes, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v < 3) return CCC_OK;
    if (!packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "packed_d must be non-NULL and 16-B aligned");
    const Sp3Layout L = sp3_layout(n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_sparse3_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    CCC_CUDA(ccc::launch_expand_sparse(packed_d, n_v, n_f, gamma, reinterpret_cast<int8_t*>(ws + L.X),
                                       reinterpret_cast<int32_t*>(ws + L.s), reinterpret_cast<int32_t*>(ws + L.c),
                                       reinterpret_cast<double*>(ws + L.w), sms, (cudaStream_t)stream),
             "expand_sparse launch");
    g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_3way_sparse_stage(int64_t n_v, int64_t n_f, double gamma, int64_t n_stages, int64_t stage,
                                 uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                                 void* ws_d, size_t ws_bytes, void* scratch_d, size_t scratch_bytes,
                                 void* stream) {
    (void)gamma;   // the weights were formed by ccc_3way_sparse_prepare
    (void)scratch_d;
    (void)scratch_bytes;   // kept for ABI stability; the single-pass kernel stores no forms
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    int64_t rng[4];
    CCC_CHECK(ccc_stage_range(n_v, n_stages, stage, rng));
    if (n_v < 3 || rng[3] == 0) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    const Sp3Layout L = sp3_layout(n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_sparse3_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    const int64_t k_pad = kpad_of(n_f);
    const int8_t* X = reinterpret_cast<const int8_t*>(ws + L.X);
    const int64_t rows = 2 * ((n_v + 15) / 16 * 16);
    CUtensorMap tmS, tmB;
    CCC_CHECK(make_tmap(&tmS, X, rows, k_pad, 64));    // 64 X rows = 32 m's x {n, v}
    CCC_CHECK(make_tmap(&tmB, X, rows, k_pad, 128));   // 128 X rows = 64 n's x {n, v}
    int64_t units = 0;
    CCC_CUDA(ccc::launch_tally3_sparse(tmS, tmB, X, reinterpret_cast<const double*>(ws + L.w), n_v, rng[0], rng[1],
                                       rng[2], k_pad, out_flags, tallies_d, ccc_d,
                                       reinterpret_cast<unsigned long long*>(checksum_d), sms,
                                       (cudaStream_t)stream, &units),
             "tally3 sparse launch");
    if (units) g_launches = 1;
    return CCC_OK;
}

// ---------------------------------------------------------------- f4(ii): paper's route
namespace {
struct PapLayout {
    size_t N = 0, s = 0, w = 0, M = 0, cnt = 0, mx = 0, total = 0;
};
PapLayout pap_layout(int64_t n_v, int64_t n_f) {
    PapLayout L;
    size_t off = 0;
    const size_t mat = al256((size_t)n_v * (size_t)kpad_of(n_f));
    L.N = off;   // rows padded to a multiple of 8 (the B operand's 4-D view)
    off += al256((size_t)((n_v + 7) / 8 * 8) * (size_t)kpad_of(n_f));
    L.s = off;
    off += al256((size_t)n_v * 4);
    L.w = off;
    off += al256((size_t)n_v * 16);
    L.M = off;                      // 3 class masks, contiguous [3][n_v][K_pad]
    off += al256(3 * (size_t)n_v * (size_t)kpad_of(n_f));
    L.cnt = off;                    // [3][n_v]
    off += al256(3 * (size_t)n_v * 4);
    L.mx = off;                     // [3][n_v][n_v] masked marginals
    off += al256(3 * (size_t)n_v * (size_t)n_v * 4);
    L.total = off + 256;
    return L;
}
}  // namespace

size_t ccc_3way_paper_workspace_bytes(int64_t n_v, int64_t n_f) {
    if (n_v < 0 || n_f < 1) return 0;
    return pap_layout(n_v, n_f).total;
}

size_t ccc_3way_paper_scratch_bytes(int64_t n_v, int64_t n_stages, int64_t stage) {
    int64_t rng[4];
    if (n_v < 3 || ccc_stage_range(n_v, n_stages, stage, rng) != CCC_OK) return 0;
    return (size_t)2 * (size_t)rng[3] * sizeof(uint32_t);
}

ccc_status ccc_3way_paper_prepare(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma, void* ws_d,
                                  size_t ws_bytes, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v < 3) return CCC_OK;
    if (!packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "packed_d must be non-NULL and 16-B aligned");
    const PapLayout L = pap_layout(n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_3way_paper_workspace_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    cudaStream_t st = (cudaStream_t)stream;
    int8_t* N = reinterpret_cast<int8_t*>(ws + L.N);
    int32_t* s = reinterpret_cast<int32_t*>(ws + L.s);
    double* w = reinterpret_cast<double*>(ws + L.w);
    int8_t* M = reinterpret_cast<int8_t*>(ws + L.M);
    CCC_CUDA(ccc::launch_expand(packed_d, n_v, n_f, gamma, N, s, w, sms, st), "expand launch");
    CCC_CUDA(ccc::launch_expand_masks(packed_d, n_v, n_f, M, reinterpret_cast<int32_t*>(ws + L.cnt), sms, st),
             "expand_masks launch");
    g_launches = 2;
    // masked marginals Mx_xi[p][x] = sum_{q: v_pq in xi} n_xq: the tally GEMM of the mask
    // rows against N over the full square (no records, raw G out)
    const size_t mat = (size_t)n_v * (size_t)kpad_of(n_f);
    for (int x = 0; x < 3; ++x)
        CCC_CHECK(block_impl(M + x * mat, s, w, n_v, 0, 0, n_v, N, s, w, n_v, 0, 0, n_f, gamma, 0, nullptr,
                             nullptr, nullptr, reinterpret_cast<int32_t*>(ws + L.mx) + (size_t)x * n_v * n_v, n_v,
                             nullptr, st, sms));
    return CCC_OK;
}

ccc_status ccc_3way_paper_stage(int64_t n_v, int64_t n_f, double gamma, int64_t n_stages, int64_t stage,
                                uint32_t out_flags, uint32_t* tallies_d, void* ccc_d, uint64_t* checksum_d,
                                void* ws_d, size_t ws_bytes, void* scratch_d, size_t scratch_bytes, void* stream) {
    (void)gamma;   // the weights were formed by ccc_3way_paper_prepare
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    int64_t rng[4];
    CCC_CHECK(ccc_stage_range(n_v, n_stages, stage, rng));
    if (n_v < 3 || rng[3] == 0) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    const PapLayout L = pap_layout(n_v, n_f);
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_3way_paper_workspace_bytes)");
    if (!scratch_d || !aligned(scratch_d, 16) || scratch_bytes < (size_t)2 * (size_t)rng[3] * 4)
        return fail(CCC_ERR_WORKSPACE, "scratch too small (see ccc_3way_paper_scratch_bytes)");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    const int64_t k_pad = kpad_of(n_f);
    const size_t mat = (size_t)n_v * (size_t)k_pad;
    const int8_t* N = reinterpret_cast<const int8_t*>(ws + L.N);
    const int32_t* s = reinterpret_cast<const int32_t*>(ws + L.s);
    const double* w = reinterpret_cast<const double*>(ws + L.w);
    const int8_t* M = reinterpret_cast<const int8_t*>(ws + L.M);
    const int32_t* mx = reinterpret_cast<const int32_t*>(ws + L.mx);
    CUtensorMap tm, tmB;
    int32_t permb = 0;
    CCC_CHECK(make_tmap(&tm, N, n_v, k_pad, 128));
    CCC_CHECK(make_tmap_b3(&tmB, N, n_v, (n_v + 7) / 8 * 8, k_pad, &permb));
    for (int x = 0; x < 3; ++x) {   // the three masked pivot GEMMs (the paper's 3 mGEMM3)
        ccc::Tally3Args a{};
        a.bp = ccc::Blk3{M + x * mat, s, w, n_v, 0};   // pivot rows: the class-xi mask
        a.bm = a.bn = ccc::Blk3{N, s, w, n_v, 0};
        a.p_lo = rng[0];
        a.p_hi = rng[1];
        a.m_hi = a.n_hi = n_v;
        a.same_pm = a.same_mn = 1;
        a.ppair = 1;
        a.ldG = n_v;
        a.rec_base = rng[2];
        a.k_pad = k_pad;
        a.n_f = (int32_t)n_f;
        a.k_blocks = (int32_t)(k_pad / ccc::kBK);
        a.out_flags = (int32_t)out_flags;
        a.tallies = tallies_d;
        a.ccc = ccc_d;
        a.checksum = reinterpret_cast<unsigned long long*>(checksum_d);
        a.forms = static_cast<uint32_t*>(scratch_d);
        a.form_stride = rng[3];
        a.form_self = x;
        a.mode = x < 2 ? 1 : 3;
        for (int y = 0; y < 3; ++y) a.mx[y] = mx + (size_t)y * n_v * n_v;
        a.mcnt = reinterpret_cast<const int32_t*>(ws + L.cnt);
        int64_t units = 0;
        a.permb = permb;
        CCC_CUDA(ccc::launch_tally3(tm, tmB, a, sms, (cudaStream_t)stream, &units), "tally3 paper-route launch");
        if (units) ++g_launches;
    }
    return CCC_OK;
}

int64_t ccc_3way_unit_records(const ccc_block* bp, int64_t p_lo, int64_t p_hi,
                              const ccc_block* bm, int64_t m_lo, int64_t m_hi,
                              const ccc_block* bn, int64_t n_lo, int64_t n_hi) {
    if (!bp || !bm || !bn || p_lo < 0 || p_hi < p_lo || m_lo < 0 || m_hi < m_lo || n_lo < 0 ||
        n_hi < n_lo)
        return -1;
    const bool spm = bp->row0 == bm->row0, smn = bm->row0 == bn->row0;
    if (spm && smn) {   // one block, whole ranges for m and n: triples with p in [p_lo, p_hi)
        const int64_t nb = bp->rows;
        return c3(nb - p_lo) - c3(nb - p_hi);
    }
    if (spm) {          // pairs (p < m) of the block with p in [p_lo, p_hi), times |N|
        const int64_t nb = bp->rows;
        auto rs = [&](int64_t i) { return i * (2 * nb - i - 1) / 2; };
        return (rs(p_hi) - rs(p_lo)) * (n_hi - n_lo);
    }
    return (p_hi - p_lo) * (m_hi - m_lo) * (n_hi - n_lo);
}

ccc_status ccc_3way_unit(const ccc_block* bp, int64_t p_lo, int64_t p_hi, const ccc_block* bm,
                         int64_t m_lo, int64_t m_hi, const ccc_block* bn, int64_t n_lo,
                         int64_t n_hi, int order, const int32_t* G_d, int64_t ldG, int64_t n_f,
                         double gamma, uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                         uint64_t* checksum_d, const ccc_compact* compact, void* stream) {
    CCC_CHECK(check_compact(compact));
    g_launches = 0;
    if (!bp || !bm || !bn) return fail(CCC_ERR_INVALID_ARGUMENT, "block descriptors must not be NULL");
    CCC_CHECK(check_sizes(bp->rows, n_f));
    CCC_CHECK(check_sizes(bm->rows, n_f));
    CCC_CHECK(check_sizes(bn->rows, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (order < 0 || order > 5) return fail(CCC_ERR_INVALID_ARGUMENT, "order must be 0..5");
    if (!(0 <= p_lo && p_lo <= p_hi && p_hi <= bp->rows && 0 <= m_lo && m_lo <= m_hi &&
          m_hi <= bm->rows && 0 <= n_lo && n_lo <= n_hi && n_hi <= bn->rows))
        return fail(CCC_ERR_INVALID_ARGUMENT, "ranges must lie inside their blocks");
    const bool spm = bp->row0 == bm->row0, smn = bm->row0 == bn->row0;
    const bool spn = bp->row0 == bn->row0;
    if ((spm && bp->N != bm->N) || (smn && bm->N != bn->N))
        return fail(CCC_ERR_INVALID_ARGUMENT, "blocks with equal row0 must be the same block");
    if (spn && !spm) return fail(CCC_ERR_INVALID_ARGUMENT, "pivot and column block equal but row block differs");
    if (smn && !(m_lo == 0 && n_lo == 0 && m_hi == bm->rows && n_hi == bn->rows))
        return fail(CCC_ERR_INVALID_ARGUMENT, "same row/column block needs whole ranges");
    if (spm && !smn && !(m_lo == 0 && m_hi == bm->rows))
        return fail(CCC_ERR_INVALID_ARGUMENT, "same pivot/row block needs the whole row range");
    {
        // slot position of each role under `order` (include/ccc.h: 0 pmn, 1 pnm, 2 mpn,
        // 3 mnp, 4 npm, 5 nmp).  A shared block enumerates p < m (m < n) only, so the
        // order must place those roles in that order or the keys are not canonical.
        static const int pos_p[6] = {0, 0, 1, 2, 1, 2}, pos_m[6] = {1, 2, 0, 0, 2, 1},
                         pos_n[6] = {2, 1, 2, 1, 0, 0};
        if (spm && pos_p[order] > pos_m[order])
            return fail(CCC_ERR_INVALID_ARGUMENT, "pivot and row block shared: order must put p before m");
        if (smn && pos_m[order] > pos_n[order])
            return fail(CCC_ERR_INVALID_ARGUMENT, "row and column block shared: order must put m before n");
    }
    const int64_t recs = ccc_3way_unit_records(bp, p_lo, p_hi, bm, m_lo, m_hi, bn, n_lo, n_hi);
    if (recs == 0) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!G_d || ldG <= 0) return fail(CCC_ERR_INVALID_ARGUMENT, "G_d must be a [ldG][ldG] pairwise G");
    for (const ccc_block* b : {bp, bm, bn})
        if (!b->N || !b->s || !b->w || !aligned(b->N, 128) || b->row0 < 0 || b->row0 + b->rows > ldG)
            return fail(CCC_ERR_INVALID_ARGUMENT, "block N (128-B aligned), s, w, row0 + rows <= ldG");
    int sms;
    CCC_CHECK(check_device(&sms));
    const int64_t k_pad = kpad_of(n_f);
    ccc::Tally3Args a{};
    a.bp = ccc::Blk3{bp->N, bp->s, bp->w, bp->rows, bp->row0};
    a.bm = ccc::Blk3{bm->N, bm->s, bm->w, bm->rows, bm->row0};
    a.bn = ccc::Blk3{bn->N, bn->s, bn->w, bn->rows, bn->row0};
    a.p_lo = p_lo;
    a.p_hi = p_hi;
    a.m_lo = m_lo;
    a.m_hi = m_hi;
    a.n_lo = n_lo;
    a.n_hi = n_hi;
    a.same_pm = spm;
    a.same_mn = smn;
    a.order = order;
    a.layout = (spm && smn) ? 0 : spm ? 1 : 2;
    a.ppair = a.layout == 0;
    const int64_t nb = bp->rows;
    if (a.layout == 0) a.rec_base = c3(nb) - c3(nb - p_lo);
    else if (a.layout == 1) a.rec_base = (p_lo * (2 * nb - p_lo - 1) / 2) * (n_hi - n_lo);
    else a.rec_base = 0;
    a.G = G_d;
    a.ldG = ldG;
    a.k_pad = k_pad;
    a.n_f = (int32_t)n_f;
    a.k_blocks = (int32_t)(k_pad / ccc::kBK);
    a.out_flags = (int32_t)out_flags;
    set_exact3(a, n_f, gamma);
    a.compact = compact ? 1 : 0;
    a.cmp = to_compact(compact);
    a.tallies = tallies_d;
    a.ccc = ccc_d;
    a.checksum = reinterpret_cast<unsigned long long*>(checksum_d);
    CUtensorMap tmA, tmB;
    CCC_CHECK(make_tmap(&tmA, bm->N, bm->rows, k_pad, 128));
    // a caller's block: the permuted view only when its rows are a multiple of 8 and every
    // column tile starts on a multiple of 8 (tiles start at n_lo + 256 K)
    CCC_CHECK(make_tmap_b3(&tmB, bn->N, bn->rows, n_lo % 8 == 0 ? bn->rows : 0, k_pad, &a.permb));
    int64_t units = 0;
    CCC_CUDA(ccc::launch_tally3(tmA, tmB, a, sms, (cudaStream_t)stream, &units), "tally3 launch");
    if (units) g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_3way(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                    uint32_t out_flags, int64_t n_stages, int64_t stage, uint32_t* tallies_d,
                    void* ccc_d, uint64_t* checksum_d, void* ws_d, size_t ws_bytes,
                    const ccc_compact* compact, void* stream) {
    CCC_CHECK(check_compact(compact));
    if (n_v >= 3) CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    CCC_CHECK(ccc_3way_prepare(packed_d, n_v, n_f, gamma, ws_d, ws_bytes, stream));
    const int64_t n1 = g_launches;
    CCC_CHECK(ccc_3way_stage(n_v, n_f, gamma, n_stages, stage, out_flags, tallies_d, ccc_d, checksum_d,
                             ws_d, ws_bytes, compact, stream));
    g_launches += n1;
    return CCC_OK;
}

// ----------------------------------------------------------------------------- e2e
static const int64_t kBandRecords = 32ll << 20;  // records per output band buffer

struct E2eLayout {
    size_t codes = 0, packed = 0, ws = 0, ck = 0, band_t[2] = {0, 0}, band_c[2] = {0, 0};
    size_t total = 0;
    int64_t band_cap = 0;
};

static E2eLayout e2e_layout(int64_t n_v, int64_t n_f, uint32_t flags) {
    E2eLayout L;
    size_t off = 0;
    L.codes = off;
    off += al256((size_t)n_v * n_f);
    L.packed = off;
    off += al256((size_t)n_v * pstride_of(n_f));
    L.ws = off;
    off += al256(ws_layout(2, n_v, n_f).total);
    L.ck = off;
    off += 256;
    const int64_t recs = c2(n_v);
    L.band_cap = std::min<int64_t>(recs, kBandRecords);
    const int64_t min_cap = 128 * std::max<int64_t>(n_v - 1, 1);  // one 128-row band
    if (L.band_cap < std::min<int64_t>(recs, min_cap)) L.band_cap = std::min<int64_t>(recs, min_cap);
    const size_t cb = (flags & CCC_OUT_CCC_F64) ? 32 : (flags & CCC_OUT_CCC_F32) ? 16 : 0;
    for (int b = 0; b < 2; ++b) {
        L.band_t[b] = off;
        if (flags & CCC_OUT_TALLY) off += al256((size_t)L.band_cap * 16);
        L.band_c[b] = off;
        off += al256((size_t)L.band_cap * cb);
    }
    L.total = off + 256;
    return L;
}

size_t ccc_e2e_workspace_bytes(int64_t n_v, int64_t n_f, uint32_t out_flags) {
    if (n_v < 0 || n_f < 1) return 0;
    return e2e_layout(n_v, n_f, out_flags).total;
}

ccc_status ccc_2way_host(const uint8_t* codes_h, int64_t n_v, int64_t n_f, double gamma,
                         uint32_t out_flags, uint32_t* tallies_h, void* ccc_h,
                         uint64_t* checksum_h, void* dev_ws_d, size_t dev_ws_bytes,
                         void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (n_v < 2) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_h, ccc_h, checksum_h));
    if (!codes_h) return fail(CCC_ERR_INVALID_ARGUMENT, "codes_h must not be NULL");
    const E2eLayout L = e2e_layout(n_v, n_f, out_flags);
    if (!dev_ws_d || !aligned(dev_ws_d, 256))
        return fail(CCC_ERR_INVALID_ARGUMENT, "dev_ws_d must be 256-B aligned");
    if (dev_ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "device workspace too small");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* base = static_cast<uint8_t*>(dev_ws_d);
    uint8_t* codes = base + L.codes;
    const WsLayout W = ws_layout(2, n_v, n_f);
    int8_t* N = reinterpret_cast<int8_t*>(base + L.ws + W.N);
    int32_t* s = reinterpret_cast<int32_t*>(base + L.ws + W.s);
    double* w = reinterpret_cast<double*>(base + L.ws + W.w);
    uint64_t* ck = reinterpret_cast<uint64_t*>(base + L.ck);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t cbytes = (out_flags & CCC_OUT_CCC_F64) ? 8 : 4;
    const bool want_c = out_flags & (CCC_OUT_CCC_F64 | CCC_OUT_CCC_F32);

    CCC_CUDA(cudaMemcpyAsync(codes, codes_h, (size_t)n_v * n_f, cudaMemcpyHostToDevice, st), "H2D codes");
    // unpacked codes straight to the operand (no 2-bit intermediate on one GPU)
    CCC_CUDA(ccc::launch_expand_codes(codes, n_v, n_f, gamma, N, s, w, sms, st), "expand_codes launch");
    int64_t launches = 1;
    if (out_flags & CCC_OUT_CHECKSUM) CCC_CUDA(cudaMemsetAsync(ck, 0, 16, st), "memset");

    cudaStream_t cs = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
    ccc_status rc = CCC_OK;
    auto cleanup = [&]() {
        for (int b = 0; b < 2; ++b) {
            if (done[b]) cudaEventDestroy(done[b]);
            if (copied[b]) cudaEventDestroy(copied[b]);
        }
        if (cs) cudaStreamDestroy(cs);
    };
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(e, "stream/event create");
    }
    auto rowstart = [&](int64_t i) { return i * (2 * n_v - i - 1) / 2; };
    int64_t r0 = 0, band = 0;
    while (r0 < n_v - 1 && rc == CCC_OK) {
        // grow the band in 128-row steps while its records fit the band buffer
        int64_t r1 = std::min<int64_t>(n_v, r0 + 128);
        while (r1 < n_v && rowstart(std::min<int64_t>(n_v, r1 + 128)) - rowstart(r0) <= L.band_cap)
            r1 = std::min<int64_t>(n_v, r1 + 128);
        const int64_t rec0 = rowstart(r0), nrec = rowstart(r1) - rec0;
        const int b = (int)(band & 1);
        if (band >= 2 && (e = cudaStreamWaitEvent(st, copied[b], 0)) != cudaSuccess) {
            rc = cuda_fail(e, "wait");
            break;
        }
        uint32_t* bt = reinterpret_cast<uint32_t*>(base + L.band_t[b]);
        void* bc = base + L.band_c[b];
        rc = block_impl(N, s, w, n_v, 0, r0, r1, N, s, w, n_v, 0, 1, n_f, gamma, out_flags, bt, bc, ck,
                        nullptr, 0, nullptr, st, sms);
        if (rc != CCC_OK) break;
        ++launches;
        if ((e = cudaEventRecord(done[b], st)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(cs, done[b], 0)) != cudaSuccess) {
            rc = cuda_fail(e, "event");
            break;
        }
        if (out_flags & CCC_OUT_TALLY)
            e = cudaMemcpyAsync(tallies_h + 4 * rec0, bt, (size_t)nrec * 16, cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess && want_c)
            e = cudaMemcpyAsync(static_cast<uint8_t*>(ccc_h) + (size_t)rec0 * 4 * cbytes, bc,
                                (size_t)nrec * 4 * cbytes, cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess) e = cudaEventRecord(copied[b], cs);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "D2H band");
            break;
        }
        r0 = r1;
        ++band;
    }
    if (rc == CCC_OK && (out_flags & CCC_OUT_CHECKSUM)) {
        e = cudaMemcpyAsync(checksum_h, ck, 16, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H checksum");
    }
    if ((e = cudaStreamSynchronize(cs)) != cudaSuccess && rc == CCC_OK) rc = cuda_fail(e, "sync copy stream");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess && rc == CCC_OK) rc = cuda_fail(e, "sync stream");
    cleanup();
    if (rc == CCC_OK) g_launches = launches;
    return rc;
}

// ------------------------------------------------------- f2: 3-way stage streaming to host
namespace {
struct H3Layout {
    size_t codes = 0, packed = 0, ws = 0, ck = 0, st_t[2] = {0, 0}, st_c[2] = {0, 0}, total = 0;
    int64_t stage_cap = 0;
};
H3Layout h3_layout(int64_t n_v, int64_t n_f, int64_t n_stages, uint32_t flags) {
    H3Layout L;
    size_t off = 0;
    L.codes = off;
    off += al256((size_t)n_v * n_f);
    L.packed = off;
    off += al256((size_t)n_v * pstride_of(n_f));
    L.ws = off;
    off += al256(ws_layout(3, n_v, n_f).total);
    L.ck = off;
    off += 256;
    int64_t cap = 0, rng[4];
    for (int64_t st = 0; st < n_stages; ++st)
        if (ccc_stage_range(n_v, n_stages, st, rng) == CCC_OK) cap = std::max<int64_t>(cap, rng[3]);
    L.stage_cap = cap;
    const size_t cb = (flags & CCC_OUT_CCC_F64) ? 64 : (flags & CCC_OUT_CCC_F32) ? 32 : 0;
    for (int b = 0; b < 2; ++b) {
        L.st_t[b] = off;
        if (flags & CCC_OUT_TALLY) off += al256((size_t)cap * 32);
        L.st_c[b] = off;
        off += al256((size_t)cap * cb);
    }
    L.total = off + 256;
    return L;
}
}  // namespace

size_t ccc_3way_host_workspace_bytes(int64_t n_v, int64_t n_f, int64_t n_stages, uint32_t out_flags) {
    if (n_v < 3 || n_f < 1 || n_stages < 1) return 256;
    return h3_layout(n_v, n_f, n_stages, out_flags).total;
}

ccc_status ccc_3way_host(const uint8_t* codes_h, int64_t n_v, int64_t n_f, double gamma, uint32_t out_flags,
                         int64_t n_stages, uint32_t* tallies_h, void* ccc_h, uint64_t* checksum_h,
                         void* dev_ws_d, size_t dev_ws_bytes, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (n_stages < 1) return fail(CCC_ERR_INVALID_ARGUMENT, "n_stages must be >= 1");
    if (n_v < 3) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_h, ccc_h, checksum_h));
    if (!codes_h) return fail(CCC_ERR_INVALID_ARGUMENT, "codes_h must not be NULL");
    const H3Layout L = h3_layout(n_v, n_f, n_stages, out_flags);
    if (!dev_ws_d || !aligned(dev_ws_d, 256))
        return fail(CCC_ERR_INVALID_ARGUMENT, "dev_ws_d must be 256-B aligned");
    if (dev_ws_bytes < L.total) return fail(CCC_ERR_WORKSPACE, "device workspace too small");
    int sms;
    CCC_CHECK(check_device(&sms));
    uint8_t* base = static_cast<uint8_t*>(dev_ws_d);
    uint8_t* ws = base + L.ws;
    const size_t ws_bytes = ws_layout(3, n_v, n_f).total;
    uint64_t* ck = reinterpret_cast<uint64_t*>(base + L.ck);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t cbytes = (out_flags & CCC_OUT_CCC_F64) ? 8 : 4;
    const bool want_c = out_flags & (CCC_OUT_CCC_F64 | CCC_OUT_CCC_F32);
    CCC_CUDA(cudaMemcpyAsync(base + L.codes, codes_h, (size_t)n_v * n_f, cudaMemcpyHostToDevice, st), "H2D codes");
    CCC_CUDA(ccc::launch_pack(base + L.codes, n_v, n_f, base + L.packed, sms, st), "pack launch");
    CCC_CHECK(ccc_3way_prepare(base + L.packed, n_v, n_f, gamma, ws, ws_bytes, stream));
    int64_t launches = 1 + g_launches;
    if (out_flags & CCC_OUT_CHECKSUM) CCC_CUDA(cudaMemsetAsync(ck, 0, 16, st), "memset");
    cudaStream_t cs = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
    ccc_status rc = CCC_OK;
    auto cleanup = [&]() {
        for (int b = 0; b < 2; ++b) {
            if (done[b]) cudaEventDestroy(done[b]);
            if (copied[b]) cudaEventDestroy(copied[b]);
        }
        if (cs) cudaStreamDestroy(cs);
    };
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        cleanup();
        return cuda_fail(e, "stream/event create");
    }
    // stage s computes into buffer s % 2 while the copy stream drains stage s - 1 to host
    for (int64_t sg = 0; sg < n_stages && rc == CCC_OK; ++sg) {
        int64_t rng[4];
        rc = ccc_stage_range(n_v, n_stages, sg, rng);
        if (rc != CCC_OK || rng[3] == 0) continue;
        const int b = (int)(sg & 1);
        if (sg >= 2 && (e = cudaStreamWaitEvent(st, copied[b], 0)) != cudaSuccess) {
            rc = cuda_fail(e, "wait");
            break;
        }
        uint32_t* bt = reinterpret_cast<uint32_t*>(base + L.st_t[b]);
        void* bc = base + L.st_c[b];
        rc = ccc_3way_stage(n_v, n_f, gamma, n_stages, sg, out_flags, (out_flags & CCC_OUT_TALLY) ? bt : nullptr,
                            want_c ? bc : nullptr, (out_flags & CCC_OUT_CHECKSUM) ? ck : nullptr, ws, ws_bytes,
                            nullptr, stream);
        if (rc != CCC_OK) break;
        launches += g_launches;
        if ((e = cudaEventRecord(done[b], st)) != cudaSuccess || (e = cudaStreamWaitEvent(cs, done[b], 0)) != cudaSuccess) {
            rc = cuda_fail(e, "event");
            break;
        }
        const int64_t rec0 = rng[2], nrec = rng[3];
        if (out_flags & CCC_OUT_TALLY)
            e = cudaMemcpyAsync(tallies_h + 8 * rec0, bt, (size_t)nrec * 32, cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess && want_c)
            e = cudaMemcpyAsync(static_cast<uint8_t*>(ccc_h) + (size_t)rec0 * 8 * cbytes, bc, (size_t)nrec * 8 * cbytes,
                                cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess) e = cudaEventRecord(copied[b], cs);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "D2H stage");
            break;
        }
    }
    if (rc == CCC_OK && (out_flags & CCC_OUT_CHECKSUM)) {
        e = cudaMemcpyAsync(checksum_h, ck, 16, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H checksum");
    }
    if ((e = cudaStreamSynchronize(cs)) != cudaSuccess && rc == CCC_OK) rc = cuda_fail(e, "sync copy stream");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess && rc == CCC_OK) rc = cuda_fail(e, "sync stream");
    cleanup();
    if (rc == CCC_OK) g_launches = launches;
    return rc;
}

// ------------------------------------------------------------------ sparse mode (f1)
int64_t ccc_sparse_rows(int64_t n_v) { return n_v < 0 ? -1 : 2 * ((n_v + 15) / 16 * 16); }

size_t ccc_sparse_workspace_bytes(int64_t n_v, int64_t n_f) {
    if (n_v < 0 || n_f < 1) return 0;
    size_t off = al256((size_t)ccc_sparse_rows(n_v) * (size_t)kpad_of(n_f));   // X
    off += al256((size_t)n_v * 4) * 2;                                           // s, c
    off += al256((size_t)n_v * 16);                                              // w
    return off + 256;
}

ccc_status ccc_expand_sparse(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                             int8_t* X_d, int32_t* s_d, int32_t* c_d, double* w_d, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_sizes(n_v, n_f));
    if (n_v == 0) return CCC_OK;
    if (!packed_d || !X_d || !s_d || !c_d || !w_d || !aligned(packed_d, 16) || !aligned(X_d, 128) ||
        !aligned(s_d, 4) || !aligned(c_d, 4) || !aligned(w_d, 8))
        return fail(CCC_ERR_INVALID_ARGUMENT,
                    "packed_d (16-B), X_d (128-B), s_d, c_d, w_d must be non-NULL and aligned");
    int sms;
    CCC_CHECK(check_device(&sms));
    CCC_CUDA(ccc::launch_expand_sparse(packed_d, n_v, n_f, gamma, X_d, s_d, c_d, w_d, sms,
                                       (cudaStream_t)stream), "expand_sparse launch");
    g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_2way_sparse_block(const int8_t* X_a, const double* w_a, int64_t n_a, int64_t a_row0,
                                 int64_t a_lo, int64_t a_hi, const int8_t* X_b, const double* w_b,
                                 int64_t n_b, int64_t b_row0, int diag, int64_t n_f,
                                 uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                                 uint64_t* checksum_d, const ccc_compact* compact, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_compact(compact));
    CCC_CHECK(check_sizes(n_a, n_f));
    CCC_CHECK(check_sizes(n_b, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (!(0 <= a_lo && a_lo <= a_hi && a_hi <= n_a))
        return fail(CCC_ERR_INVALID_ARGUMENT, "need 0 <= a_lo <= a_hi <= n_a");
    if (diag && (X_a != X_b || n_a != n_b || a_row0 != b_row0))
        return fail(CCC_ERR_INVALID_ARGUMENT, "diag block needs A == B");
    if (a_row0 < 0 || b_row0 < 0 || a_row0 + n_a > CCC_MAX_NV || b_row0 + n_b > CCC_MAX_NV)
        return fail(CCC_ERR_INVALID_ARGUMENT, "global row indices out of range");
    if (a_hi == a_lo || n_b == 0) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!X_a || !X_b || !w_a || !w_b || !aligned(X_a, 128) || !aligned(X_b, 128))
        return fail(CCC_ERR_INVALID_ARGUMENT, "X_a/X_b (128-B aligned), w must be non-NULL");
    int sms;
    CCC_CHECK(check_device(&sms));
    const int64_t k_pad = kpad_of(n_f);
    CUtensorMap tmA, tmB;
    CCC_CHECK(make_tmap(&tmA, X_a, ccc_sparse_rows(n_a), k_pad, 128));
    CCC_CHECK(make_tmap(&tmB, X_b, ccc_sparse_rows(n_b), k_pad, 128));
    ccc::Tally2Args a{};
    const int64_t v_lo16 = a_lo / 16 * 16, v_hi16 = (a_hi + 15) / 16 * 16;
    a.sparse = 1;
    a.a_lo = 2 * v_lo16;                 // scheduler / TMA coordinates: rows of X
    a.nA = 2 * (v_hi16 - v_lo16);
    a.nB = ccc_sparse_rows(n_b);
    a.v_lo = a_lo;                       // records: vectors
    a.v_hi = a_hi;
    a.nBv = n_b;
    a.a_row0 = a_row0;
    a.b_row0 = b_row0;
    a.diag = diag ? 1 : 0;
    a.n_f = (int32_t)n_f;
    a.k_blocks = (int32_t)(k_pad / ccc::kBK);
    a.out_flags = (int32_t)out_flags;
    a.w_a = w_a;
    a.w_b = w_b;
    a.tallies = tallies_d;
    a.ccc = ccc_d;
    a.checksum = reinterpret_cast<unsigned long long*>(checksum_d);
    a.rec_row_base = diag ? (a_lo * (2 * n_b - a_lo - 1)) / 2 : 0;
    a.sup_rows = 2048;
    a.sup_cols = 2048;
    a.compact = compact ? 1 : 0;
    a.cmp = to_compact(compact);
    int64_t tiles = 0;
    CCC_CUDA(ccc::launch_tally2(tmA, tmB, a, sms, (cudaStream_t)stream, &tiles), "tally2 sparse launch");
    if (tiles) g_launches = 1;
    return CCC_OK;
}

ccc_status ccc_2way_sparse(const uint8_t* packed_d, int64_t n_v, int64_t n_f, double gamma,
                           uint32_t out_flags, uint32_t* tallies_d, void* ccc_d,
                           uint64_t* checksum_d, void* ws_d, size_t ws_bytes,
                           const ccc_compact* compact, void* stream) {
    g_launches = 0;
    CCC_CHECK(check_compact(compact));
    CCC_CHECK(check_sizes(n_v, n_f));
    if (out_flags & ~15u) return fail(CCC_ERR_INVALID_ARGUMENT, "unknown out_flags bits");
    if (n_v < 2) return CCC_OK;
    CCC_CHECK(check_outputs(out_flags, tallies_d, ccc_d, checksum_d));
    if (!packed_d || !aligned(packed_d, 16))
        return fail(CCC_ERR_INVALID_ARGUMENT, "packed_d must be non-NULL and 16-B aligned");
    if (!ws_d || !aligned(ws_d, 256)) return fail(CCC_ERR_INVALID_ARGUMENT, "ws_d must be 256-B aligned");
    if (ws_bytes < ccc_sparse_workspace_bytes(n_v, n_f))
        return fail(CCC_ERR_WORKSPACE, "workspace too small (see ccc_sparse_workspace_bytes)");
    uint8_t* ws = static_cast<uint8_t*>(ws_d);
    size_t off = 0;
    int8_t* X = reinterpret_cast<int8_t*>(ws);
    off += al256((size_t)ccc_sparse_rows(n_v) * (size_t)kpad_of(n_f));
    int32_t* sv = reinterpret_cast<int32_t*>(ws + off);
    off += al256((size_t)n_v * 4);
    int32_t* cv = reinterpret_cast<int32_t*>(ws + off);
    off += al256((size_t)n_v * 4);
    double* w = reinterpret_cast<double*>(ws + off);
    CCC_CHECK(ccc_expand_sparse(packed_d, n_v, n_f, gamma, X, sv, cv, w, stream));
    CCC_CHECK(ccc_2way_sparse_block(X, w, n_v, 0, 0, n_v, X, w, n_v, 0, 1, n_f, out_flags,
                                    tallies_d, ccc_d, checksum_d, compact, stream));
    g_launches += 1;
    return CCC_OK;
}

}  // extern "C"
