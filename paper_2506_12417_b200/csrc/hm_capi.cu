// C ABI of libharmoe.so (declared in include/harmoe.h) + host utilities:
// error state, SM count, TMA descriptor encoding and the K6 fetch primitive.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HM_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return HM_OK;
}

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static PFN_cuStreamWriteValue32_v11070 g_write32 = nullptr;
static PFN_cuMemGetAddressRange_v3020 g_addr_range = nullptr;
static PFN_cuStreamWaitValue32_v11070 g_wait32 = nullptr;
static std::once_flag g_driver_once;

static void load_driver_entry_points() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  fn = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_write32 = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(fn);
  fn = nullptr;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_addr_range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
  fn = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_wait32 = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(fn);
}

int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                      uint32_t box_cols) {
  std::call_once(g_driver_once, load_driver_entry_points);
  if (g_encode == nullptr) return set_error(HM_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return set_error(HM_EINVAL, "TMA base must be 16-byte aligned");
  if ((cols * 2) % 16 != 0) return set_error(HM_EINVAL, "TMA row pitch must be a multiple of 16 bytes");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(HM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HM_OK;
}

int launch_hist_scan(const int32_t*, int, int, int, int32_t*, int32_t*, cudaStream_t);
int launch_schedule(const int32_t*, const int32_t*, int, int, int, int, int32_t*, int32_t*, int32_t*, cudaStream_t);
int launch_rebalance(int32_t*, int, int, int, int32_t*, int32_t*, cudaStream_t);
int launch_schedule_batched(const int32_t*, const int32_t*, int, int, int, int, int, int32_t*, int32_t*, int32_t*,
                            cudaStream_t);
int read_plan_phases(long long*);
int launch_plan(const int32_t*, int, const int32_t*, const int32_t*, int, int, int, int, int, int, int32_t*, int32_t*,
                int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int32_t*, int,
                cudaStream_t, int32_t* = nullptr, int32_t* = nullptr, int32_t* = nullptr);
int launch_dispatch_push_ordered(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*,
                                 const int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int, int,
                                 int, int, const unsigned long long*, const unsigned long long*,
                                 const unsigned long long*, int32_t*, int32_t*, uint32_t*, cudaStream_t);
int launch_layout(const int32_t*, const int32_t*, int, int, int, int, int32_t*, int32_t*, int32_t*, int32_t*,
                  int32_t*, int32_t*, int, cudaStream_t);
int launch_permute(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, int,
                   int, int, int, int, int, int, void*, int32_t*, int32_t*, cudaStream_t);
int launch_combine(const void*, const int32_t*, const float*, int, int, int, const void*, void*, cudaStream_t);
int launch_ep_offsets(const int32_t*, int, int, int, int32_t*, int32_t*, cudaStream_t);
int launch_dispatch_push(const void*, const int32_t*, const int32_t*, const int32_t*, const int32_t*, const int32_t*,
                         const int32_t*, int, int, int, int, int, int, const unsigned long long*,
                         const unsigned long long*, int32_t*, cudaStream_t);
int launch_fetch_experts(const int32_t*, const int32_t*, const unsigned long long*, const unsigned long long*, size_t,
                         size_t, void*, void*, int, int, int32_t*, int32_t*, int32_t*, int, int, int, cudaStream_t);

// Flag publish by a kernel (used when stream memory operations are unavailable): the stream
// order makes every earlier kernel's writes complete first; the system-scope release orders
// them before the flag for a consumer on another GPU (peer flags over NVLink).
__global__ void publish_flag_kernel(int32_t* flag, int epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

}  // namespace hm

using namespace hm;

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int hm_version(void) { return 1; }

const char* hm_last_error(void) { return hm::g_err; }

int hm_num_sms(void) { return num_sms(); }

int hm_gemm_tile_m(void) { return 128; }

int hm_gemm_resident_pairs(int epilogue, int gather) {
  const int n = gemm_resident_pairs(epilogue, gather != 0);
  if (n < 0) return set_error(HM_EINVAL, "gemm_resident_pairs: unknown epilogue");
  return n;
}

int hm_router_topk(const void* x, const void* wg, const float* bias, int n_ranks, int tokens_per_rank, int d, int E,
                   int k, int renormalize, int32_t* topk_idx, float* topk_w, int32_t* tile_hist, int32_t* lrank,
                   void* stream) {
  return launch_router(x, wg, bias, n_ranks, tokens_per_rank, d, E, k, renormalize, topk_idx, topk_w, tile_hist,
                       lrank, as_stream(stream));
}

int hm_hist_scan(const int32_t* tile_hist, int n_ranks, int tiles_per_rank, int E, int32_t* hist, int32_t* tile_off,
                 void* stream) {
  return launch_hist_scan(tile_hist, n_ranks, tiles_per_rank, E, hist, tile_off, as_stream(stream));
}

int hm_schedule(const int32_t* m_all, const int32_t* home, int G, int E, int q, int rebalance, int32_t* S,
                int32_t* iters, int32_t* loads, void* stream) {
  return launch_schedule(m_all, home, G, E, q, rebalance, S, iters, loads, as_stream(stream));
}

int hm_plan(const int32_t* tile_hist, int tiles_per_rank, const int32_t* m_all_in, const int32_t* home, int G, int E,
            int q, int rebalance, int mode, int me, int32_t* m_all_out, int32_t* tile_off, int32_t* S, int32_t* iters,
            int32_t* loads, int32_t* slot_base, int32_t* segs, int32_t* n_seg, int32_t* mtile_prefix, int32_t* fetch,
            int32_t* n_fetch, int cache_slots, void* stream) {
  return launch_plan(tile_hist, tiles_per_rank, m_all_in, home, G, E, q, rebalance, mode, me, m_all_out, tile_off, S,
                     iters, loads, slot_base, segs, n_seg, mtile_prefix, fetch, n_fetch, cache_slots,
                     as_stream(stream));
}

int hm_plan_dispatch(const int32_t* m_all_in, const int32_t* home, int G, int E, int q, int rebalance, int me,
                     int32_t* S, int32_t* iters, int32_t* loads, int32_t* slot_base, int32_t* segs, int32_t* n_seg,
                     int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch, int cache_slots, int32_t* push_items,
                     int32_t* push_cprefix, int32_t* push_ebase, void* stream) {
  if (push_items == nullptr) return set_error(HM_EINVAL, "plan_dispatch: push_items is required");
  return launch_plan(nullptr, 0, m_all_in, home, G, E, q, rebalance, HM_LAYOUT_EP_EXPERT, me, nullptr, nullptr, S,
                     iters, loads, slot_base, segs, n_seg, mtile_prefix, fetch, n_fetch, cache_slots,
                     as_stream(stream), push_items, push_cprefix, push_ebase);
}

int hm_schedule_batched(const int32_t* m_all, const int32_t* home, int B, int G, int E, int q, int rebalance,
                        int32_t* S, int32_t* iters, int32_t* loads, void* stream) {
  return launch_schedule_batched(m_all, home, B, G, E, q, rebalance, S, iters, loads, as_stream(stream));
}

int hm_rebalance(int32_t* S, int G, int E, int q, int32_t* iters, int32_t* loads, void* stream) {
  return launch_rebalance(S, G, E, q, iters, loads, as_stream(stream));
}

int hm_dispatch_layout(const int32_t* S, const int32_t* home, int G, int E, int mode, int me, int32_t* slot_base,
                       int32_t* segs, int32_t* n_seg, int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch,
                       int cache_slots, void* stream) {
  return launch_layout(S, home, G, E, mode, me, slot_base, segs, n_seg, mtile_prefix, fetch, n_fetch, cache_slots,
                       as_stream(stream));
}

int hm_permute(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
               const int32_t* S, const int32_t* slot_base, int n_ranks, int tokens_per_rank, int src_rank_base, int G,
               int E, int k, int d, void* out, int32_t* pos, int32_t* inv, void* stream) {
  return launch_permute(x, topk_idx, lrank, tile_off, S, slot_base, n_ranks, tokens_per_rank, src_rank_base, G, E, k,
                        d, out, pos, inv, as_stream(stream));
}

int hm_grouped_gemm(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K, const int32_t* segs,
                    const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue, void* out,
                    const int32_t* row_map, const int32_t* a_gather, int a_gather_div, const int32_t* slot_ready,
                    int ready_from_slot, int epoch, int32_t* slot_done, const hm_fetch_plan* fetch, void* stream) {
  return launch_grouped_gemm(A, a_rows, W, w_rows, N, K, segs, n_seg, mtile_prefix, epilogue, out, row_map, a_gather,
                             a_gather_div, slot_ready, ready_from_slot, epoch, as_stream(stream), nullptr, nullptr, 0,
                             slot_done, fetch);
}

int hm_grouped_gemm_swap(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                         const int32_t* segs, const int32_t* n_seg, int epilogue, void* out, const int32_t* row_map,
                         const float* topk_w, const void* residual, void* y, void* stream) {
  const CombineFuse cf{topk_w, residual, y, nullptr, 1};
  return launch_grouped_gemm_swap(A, a_rows, W, w_rows, N, K, segs, n_seg, epilogue, out, row_map,
                                  y != nullptr ? &cf : nullptr, as_stream(stream));
}

int hm_grouped_gemm_combine(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                            const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, void* Y,
                            const int32_t* row_map, const float* topk_w, int k, const void* residual, void* y,
                            uint32_t* counters, void* stream) {
  if (y == nullptr || (Y == nullptr && k != 1))
    return set_error(HM_EINVAL, "grouped_gemm_combine: y (and Y unless k == 1) are required");
  const CombineFuse cf{topk_w, residual, y, counters, k};
  return launch_grouped_gemm(A, a_rows, W, w_rows, N, K, segs, n_seg, mtile_prefix, 0 /* STORE */, Y, row_map,
                             nullptr, 1, nullptr, 0, 0, as_stream(stream), nullptr, nullptr, 0, nullptr, nullptr,
                             &cf);
}

int hm_grouped_gemm_remote(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                           const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue,
                           const uint64_t* out_ptrs, const int32_t* out_split, int n_out, const int32_t* row_map,
                           const int32_t* slot_ready, int ready_from_slot, int epoch, int32_t* slot_done,
                           const hm_fetch_plan* fetch, void* stream) {
  if (out_ptrs == nullptr) return set_error(HM_EINVAL, "grouped_gemm_remote: out_ptrs is required");
  return launch_grouped_gemm(A, a_rows, W, w_rows, N, K, segs, n_seg, mtile_prefix, epilogue, nullptr, row_map,
                             nullptr, 1, slot_ready, ready_from_slot, epoch, as_stream(stream),
                             reinterpret_cast<const unsigned long long*>(out_ptrs), out_split, n_out, slot_done,
                             fetch);
}

int hm_grouped_gemm_arrive(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                           const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue,
                           void* out, const int32_t* slot_ready, int ready_from_slot, int epoch, int32_t* slot_done,
                           const hm_fetch_plan* fetch, const int32_t* a_arrive, int pdl, void* stream) {
  if (a_arrive == nullptr) return set_error(HM_EINVAL, "grouped_gemm_arrive: a_arrive is required");
  return launch_grouped_gemm(A, a_rows, W, w_rows, N, K, segs, n_seg, mtile_prefix, epilogue, out, nullptr, nullptr, 1,
                             slot_ready, ready_from_slot, epoch, as_stream(stream), nullptr, nullptr, 0, slot_done,
                             fetch, nullptr, a_arrive, pdl);
}

int hm_dispatch_push_ordered(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
                             const int32_t* S, const int32_t* slot_base, const int32_t* push_items,
                             const int32_t* push_cprefix, const int32_t* push_ebase, int tokens, int me, int G, int E,
                             int k, int d, const uint64_t* dst_rows, const uint64_t* dst_tok,
                             const uint64_t* dst_arrive, int32_t* order, int32_t* pos, uint32_t* sync, void* stream) {
  return launch_dispatch_push_ordered(x, topk_idx, lrank, tile_off, S, slot_base, push_items, push_cprefix, push_ebase,
                                      tokens, me, G, E, k, d, reinterpret_cast<const unsigned long long*>(dst_rows),
                                      reinterpret_cast<const unsigned long long*>(dst_tok),
                                      reinterpret_cast<const unsigned long long*>(dst_arrive), order, pos, sync,
                                      as_stream(stream));
}

int hm_ep_offsets(const int32_t* S, int G, int E, int me, int32_t* dst_delta, int32_t* recv_split, void* stream) {
  return launch_ep_offsets(S, G, E, me, dst_delta, recv_split, as_stream(stream));
}

int hm_dispatch_push(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
                     const int32_t* S, const int32_t* slot_base, const int32_t* dst_delta, int tokens, int me, int G,
                     int E, int k, int d, const uint64_t* dst_rows, const uint64_t* dst_tok, int32_t* pos,
                     void* stream) {
  return launch_dispatch_push(x, topk_idx, lrank, tile_off, S, slot_base, dst_delta, tokens, me, G, E, k, d,
                              reinterpret_cast<const unsigned long long*>(dst_rows),
                              reinterpret_cast<const unsigned long long*>(dst_tok), pos, as_stream(stream));
}

int hm_fetch_experts(const int32_t* fetch, const int32_t* n_fetch, const uint64_t* src_in, const uint64_t* src_out,
                     size_t in_bytes, size_t out_bytes, void* dst_in, void* dst_out, int first_slot, int n_slots,
                     int32_t* ready_in, int32_t* ready_out, int32_t* counters, int n_counters, int value, int ctas,
                     void* stream) {
  return launch_fetch_experts(fetch, n_fetch, reinterpret_cast<const unsigned long long*>(src_in),
                              reinterpret_cast<const unsigned long long*>(src_out), in_bytes, out_bytes, dst_in,
                              dst_out, first_slot, n_slots, ready_in, ready_out, counters, n_counters, value, ctas,
                              as_stream(stream));
}

int hm_stream_signal(void* const* flags, int n, uint32_t value, void* stream) {
  std::call_once(g_driver_once, load_driver_entry_points);
  if (n < 0 || (n > 0 && flags == nullptr)) return set_error(HM_EINVAL, "stream_signal: bad flag list");
  cudaStream_t s = as_stream(stream);
  // Per device: cleared once the driver refuses a stream write to a VALID address (e.g. peer
  // memory on some driver / topology), after which flags are published by a kernel.  A refusal
  // for an address that is not mapped at all stays an error (a bad flag pointer must not turn
  // into an illegal-address fault inside the fallback kernel).
  static std::atomic<int> memops_refused[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& refused = memops_refused[(dev >= 0 && dev < 64) ? dev : 0];
  for (int i = 0; i < n; ++i) {
    if (g_write32 != nullptr && refused.load(std::memory_order_relaxed) == 0) {
      const CUresult r = g_write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flags[i]),
                                   (cuuint32_t)value, CU_STREAM_WRITE_VALUE_DEFAULT);
      if (r == CUDA_ERROR_NOT_SUPPORTED || r == CUDA_ERROR_INVALID_VALUE) {
        CUdeviceptr base = 0;
        size_t size = 0;
        if (g_addr_range == nullptr ||
            g_addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(flags[i])) != CUDA_SUCCESS)
          return set_error(HM_EINVAL, "stream_signal: flag address %p is not mapped on this device", flags[i]);
        refused.store(1, std::memory_order_relaxed);  // valid address: fall back to the kernel publish
      } else if (r != CUDA_SUCCESS) {
        return set_error(HM_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
      } else {
        continue;
      }
    }
    {
      publish_flag_kernel<<<1, 1, 0, s>>>(reinterpret_cast<int32_t*>(flags[i]), (int)value);
      const int rc = check_launch("stream_signal");
      if (rc) return rc;
    }
  }
  return HM_OK;
}

int hm_stream_wait(const int32_t* flags, int n, uint32_t value, void* stream) {
  std::call_once(g_driver_once, load_driver_entry_points);
  if (g_wait32 == nullptr) return set_error(HM_ECUDA, "cuStreamWaitValue32 unavailable");
  cudaStream_t s = as_stream(stream);
  for (int i = 0; i < n; ++i) {
    const CUresult r = g_wait32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flags + i),
                                (cuuint32_t)value, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return set_error(HM_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
  }
  return HM_OK;
}

int hm_fetch_expert(void* dst, const void* src, size_t bytes, int32_t* ready_flag, int epoch, void* stream) {
  std::call_once(g_driver_once, load_driver_entry_points);
  cudaStream_t s = as_stream(stream);
  if (bytes > 0) {
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s);
    if (e != cudaSuccess) return set_error(HM_ECUDA, "fetch_expert memcpy: %s", cudaGetErrorString(e));
  }
  if (ready_flag == nullptr) return HM_OK;
  if (g_write32 != nullptr) {
    const CUresult r = g_write32(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(ready_flag),
                                 (cuuint32_t)epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return set_error(HM_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
    return HM_OK;
  }
  publish_flag_kernel<<<1, 1, 0, s>>>(ready_flag, epoch);
  return check_launch("fetch_expert flag");
}

int hm_debug_plan_phases(long long* out4) { return read_plan_phases(out4); }

int hm_ipc_get_handle(const void* dev_ptr, void* handle_out, size_t* offset_out) {
  std::call_once(g_driver_once, load_driver_entry_points);
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return set_error(HM_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle_out, &h, sizeof(h));
  // the handle names the whole allocation (e.g. a caching-allocator block): report where
  // dev_ptr sits inside it so the peer can add it to the base cudaIpcOpenMemHandle returns
  if (offset_out != nullptr) {
    if (g_addr_range == nullptr) return set_error(HM_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUresult r = g_addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr));
    if (r != CUDA_SUCCESS) return set_error(HM_ECUDA, "cuMemGetAddressRange failed (%d)", (int)r);
    *offset_out = (size_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  }
  return HM_OK;
}

int hm_ipc_open(const void* handle, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return set_error(HM_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  return HM_OK;
}

int hm_ipc_close(void* dev_ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return set_error(HM_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return HM_OK;
}

int hm_combine(const void* Y, const int32_t* pos, const float* topk_w, int T, int k, int d, const void* residual,
               void* y, void* stream) {
  return launch_combine(Y, pos, topk_w, T, k, d, residual, y, as_stream(stream));
}

}  // extern "C"
