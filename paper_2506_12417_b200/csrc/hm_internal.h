// Internal host-side declarations shared by the harmoe translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/harmoe.h"

namespace hm {

enum Epilogue { kEpiStore = HM_EPI_STORE, kEpiRelu = HM_EPI_RELU, kEpiSwiGLU = HM_EPI_SWIGLU };

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
int num_sms();

// K-major bf16 2-D tensor map [rows, cols] (cols contiguous), box [box_rows, box_cols],
// SWIZZLE_128B (box_cols * 2 must be 128).  Out-of-bounds rows are zero-filled.
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                      uint32_t box_cols);

// FFN2 epilogue with the weighted combine fused in (LOCAL layout, token-major scatter):
// y[t] = (residual[t] +) sum_j w[t,j] Y[t*k+j], computed by the k-th arriving row of each
// (token, 64-column chunk); counters [T, N/64] self-reset (atomicInc wraps at k - 1).
struct CombineFuse {
  const float* w;
  const void* residual;
  void* y;  // nullptr: no fused combine
  unsigned* counters;
  int k;
};

int launch_grouped_gemm(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                        const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue,
                        void* out, const int32_t* row_map, const int32_t* a_gather, int a_gather_div,
                        const int32_t* slot_ready, int ready_from_slot, int epoch, cudaStream_t stream,
                        const unsigned long long* out_ptrs = nullptr, const int32_t* out_split = nullptr,
                        int n_out = 0, int32_t* slot_done = nullptr, const hm_fetch_plan* fetch = nullptr,
                        const CombineFuse* combine = nullptr, const int32_t* a_arrive = nullptr, int pdl = 0);

int gemm_resident_pairs(int epilogue, bool gather);
int launch_grouped_gemm_swap(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                             const int32_t* segs, const int32_t* n_seg, int epilogue, void* out, const int32_t* row_map,
                             const CombineFuse* combine, cudaStream_t stream);

int launch_router(const void* x, const void* wg, const float* bias, int n_ranks, int tokens_per_rank, int d, int E,
                  int k, int renormalize, int32_t* topk_idx, float* topk_w, int32_t* tile_hist, int32_t* lrank,
                  cudaStream_t stream);

}  // namespace hm
