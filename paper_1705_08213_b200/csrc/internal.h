// internal.h -- launchers shared between the kernel translation units and abi.cu.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace ccc {

cudaError_t launch_pack(const uint8_t* codes, int64_t n_v, int64_t n_f, uint8_t* packed,
                        int num_sms, cudaStream_t stream);
cudaError_t launch_expand(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma,
                          int8_t* N, int32_t* s, double* w, int num_sms, cudaStream_t stream);
cudaError_t launch_expand_codes(const uint8_t* codes, int64_t n_v, int64_t n_f, double gamma, int8_t* N,
                                int32_t* s, double* w, int num_sms, cudaStream_t stream);
cudaError_t launch_expand_sparse(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma,
                                 int8_t* X, int32_t* s, int32_t* c, double* w, int num_sms,
                                 cudaStream_t stream);
cudaError_t launch_expand_masks(const uint8_t* packed, int64_t n_v, int64_t n_f, int8_t* M, int32_t* cnt,
                                int num_sms, cudaStream_t stream);
int tally2_b_box_rows();  // B rows per CTA per TMA box (256 single CTA, 128 CTA pair)
int tally2_tile_rows();   // rows of a 2-way tile (256 CTA pair, 128 single CTA)
int64_t fs_total_tiles(int64_t n_v);       // tiles of the whole diag 2-way schedule
int64_t fs_block_tiles(const FsGeom& g);   // tiles of one block's 2-way schedule (f3 waves)
cudaError_t launch_fs_finish(const int32_t* slots, const int32_t* s_a, const int32_t* s_b, const FsGeom& g,
                             int64_t n_f, double gamma, int owner, int world, int64_t t_lo, int64_t t_hi,
                             uint32_t flags, uint32_t* tallies, void* ccc, unsigned long long* checksum,
                             int num_sms, cudaStream_t stream);
cudaError_t launch_tally2(const CUtensorMap& tmA, const CUtensorMap& tmB, const Tally2Args& a,
                          int num_sms, cudaStream_t stream, int64_t* n_tiles_out);
cudaError_t launch_tally3(const CUtensorMap& tmA, const CUtensorMap& tmB, const Tally3Args& a,
                          int num_sms, cudaStream_t stream, int64_t* n_units_out);

cudaError_t launch_tally3_sparse(const CUtensorMap& tmSrc, const CUtensorMap& tmB, const int8_t* X,
                                 const double* w, int64_t n_v, int64_t p_lo, int64_t p_hi, int64_t rec_base,
                                 int64_t k_pad, uint32_t out_flags, uint32_t* tallies, void* ccc,
                                 unsigned long long* checksum, int num_sms, cudaStream_t stream,
                                 int64_t* n_units_out);
cudaError_t launch_popc_2way(const uint8_t* packed, int64_t n_v, int64_t n_f, double gamma, uint32_t flags,
                             uint32_t* tallies, void* ccc, unsigned long long* checksum, int32_t* s,
                             double* w, int num_sms, cudaStream_t stream);

}  // namespace ccc
