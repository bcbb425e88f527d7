// Microbenchmark: HBM read bandwidth of TMA 2-D weight streaming in the grouped GEMM's pattern
// (box = box_rows x 64 bf16, 128-byte swizzle, k-inner walk over a row block, S-stage ring),
// no MMA: one producer thread issues, one consumer thread waits/recycles.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../paper_2506_12417_b200/csrc/hm_common.cuh"
using namespace hm;

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap tm, int row_blocks, int kblocks,
                                                    int box_rows, int stages, int hint, int rb_stride) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t box_bytes = box_rows * 64 * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * box_bytes);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int nunits = ((row_blocks - blockIdx.x + gridDim.x - 1) / gridDim.x) * kblocks;
  if (threadIdx.x == 0) {
    uint64_t pol = hint == 0 ? l2_policy_evict_first() : (hint == 1 ? l2_policy_evict_normal() : l2_policy_evict_last());
    int stage = 0; uint32_t ph = 0;
    for (int u = 0; u < nunits; ++u) {
      const int rb = blockIdx.x + (u / kblocks) * gridDim.x;
      const int kb = u % kblocks;
      mbar_wait(&empty[stage], ph ^ 1);
      mbar_arrive_expect_tx(&full[stage], box_bytes);
      tma_load_2d(smem + stage * box_bytes, &tm, &full[stage], kb * 64, rb * box_rows, pol);
      if (++stage == stages) { stage = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int stage = 0; uint32_t ph = 0;
    for (int u = 0; u < nunits; ++u) {
      mbar_wait(&full[stage], ph);
      mbar_arrive(&empty[stage]);
      if (++stage == stages) { stage = 0; ph ^= 1; }
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    void* fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return f;
}

extern "C" int stream_launch(const void* W, long rows, int K, int box_rows, int stages, int grid, int hint, void* stream) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  if (enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(W), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) return -1;
  const size_t smem = 1024 + (size_t)stages * box_rows * 128 + 2 * stages * 8;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  stream_kernel<<<grid, 64, smem, (cudaStream_t)stream>>>(tm, (int)(rows / box_rows), K / 64, box_rows, stages, hint, 0);
  return (int)cudaGetLastError();
}
