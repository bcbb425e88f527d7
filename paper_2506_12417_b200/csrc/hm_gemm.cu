// K5: grouped expert GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces the expert-compute phase the reference only models
// (moesim/engine.py:128-132 CostModel.expert_flops, engine.py:354-359 per-GPU
// execution; Alg.1 step 5).  One persistent CTA per SM walks a
// device-resident tile list built by hm_dispatch_layout (no host sync):
//
//   segment s = {row_start, nrows, wslot, expert}: rows [row_start, row_start+nrows)
//   of the token buffer A are multiplied by weight slot `wslot` (W[wslot] is
//   [N, K] K-major, i.e. nn.Linear layout).  Tiles are 128 rows x 256 columns;
//   within a segment the order is n-block-major so consecutive CTAs share the
//   A rows in L2; segments come in HarMoEny plan order (engine.py:233-234:
//   residents first, then fetched experts) so async weight fetches (K6) get the
//   longest possible compute shadow.
//
// Warp roles (192 threads): warp0 = TMA producer, warp1 = MMA issuer (one
// elected thread) + TMEM owner, warps2-5 = epilogue (TMEM -> regs -> global).
// 4-stage smem ring (48 KB/stage), 2 TMEM accumulators of 256 fp32 columns so
// the epilogue of tile i overlaps the MMAs of tile i+1.
//
// Epilogues: kEpiStore (bf16 out), kEpiRelu (Switch FFN1), kEpiSwiGLU (W13 is
// block-interleaved: within each 256-row block, rows [0,128) are gate rows and
// [128,256) the matching up rows -> 128 bf16 outputs per tile).
#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

constexpr int kBM = 128;
constexpr int kBN = 256;
constexpr int kBK = 64;
constexpr int kStages = 4;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
constexpr uint32_t kBBytes = kBN * kBK * 2;  // 32 KB
constexpr uint32_t kTmemCols = 512;
constexpr int kGemmThreads = 192;
constexpr size_t kGemmSmem = 1024 + kStages * (kABytes + kBBytes) + 256;

__device__ __forceinline__ void decode_tile(int t, int NB, const int4* __restrict__ segs,
                                            const int* __restrict__ mprefix, int n_seg, int4& seg, int& m, int& nb) {
  // largest s with mprefix[s] * NB <= t
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (mprefix[mid] * NB <= t) lo = mid;
    else hi = mid - 1;
  }
  seg = segs[lo];
  const int ms = mprefix[lo + 1] - mprefix[lo];
  const int local = t - mprefix[lo] * NB;
  nb = local / ms;
  m = local - nb * ms;
}

template <int kEpi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const int4* __restrict__ segs, const int* __restrict__ mprefix,
                        const int* __restrict__ n_seg_ptr, __nv_bfloat16* __restrict__ out, int N, int K, int ldo,
                        const int* __restrict__ slot_ready, int ready_from_slot, int epoch) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_b + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int n_seg = *n_seg_ptr;
  const int NB = N / kBN;
  const int total = n_seg > 0 ? mprefix[n_seg] * NB : 0;
  const int KB = K / kBK;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_a = l2_policy_evict_normal();
      const uint64_t pol_b = l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int4 seg;
        int m, nb;
        decode_tile(t, NB, segs, mprefix, n_seg, seg, m, nb);
        const int row0 = seg.x + m * kBM;
        const int brow = seg.z * N + nb * kBN;
        if (slot_ready != nullptr && seg.z >= ready_from_slot) {
          // K6: fetched expert weights land asynchronously; wait for this slot's epoch
          while (ld_acquire_gpu(slot_ready + seg.z) < epoch) __nanosleep(64);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kABytes + kBBytes);
          tma_load_2d(smem_a + stage * kABytes, &tmap_a, &full[stage], kb * kBK, row0, pol_a);
          tma_load_2d(smem_b + stage * kBBytes, &tmap_b, &full[stage], kb * kBK, brow, pol_b);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = make_idesc_bf16(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
        const int acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = make_sdesc_sw128(smem_u32(smem_a + stage * kABytes));
          const uint64_t b0 = make_sdesc_sw128(smem_u32(smem_b + stage * kBBytes));
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // advance 16 bf16 = 32 B along K inside the 128B swizzle atom
            umma_bf16(d_tmem, a0 + (uint64_t)(k * 2), b0 + (uint64_t)(k * 2), idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ===== epilogue: warps 2..5, TMEM lane quarter = warp % 4 =====
    const int q = warp & 3;
    const int r_in_tile = q * 32 + lane;
    int i = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
      int4 seg;
      int m, nb;
      decode_tile(t, NB, segs, mprefix, n_seg, seg, m, nb);
      const int rows = min(kBM, seg.y - m * kBM);
      const bool valid = r_in_tile < rows;
      const int64_t row = (int64_t)seg.x + m * kBM + r_in_tile;
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16);
      if constexpr (kEpi == kEpiSwiGLU) {
        __nv_bfloat16* orow = out + row * ldo + nb * (kBN / 2);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(taddr + c * 32, g);
          tmem_ld_32x32b_x32(taddr + 128 + c * 32, u);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float g0 = __uint_as_float(g[2 * j]), g1 = __uint_as_float(g[2 * j + 1]);
            float u0 = __uint_as_float(u[2 * j]), u1 = __uint_as_float(u[2 * j + 1]);
            float h0 = g0 / (1.0f + __expf(-g0)) * u0;
            float h1 = g1 / (1.0f + __expf(-g1)) * u1;
            pk[j] = pack_bf16x2(h0, h1);
          }
          if (valid) {
#pragma unroll
            for (int v = 0; v < 4; ++v)
              st_global_v4(orow + c * 32 + v * 8, pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
          }
        }
      } else {
        __nv_bfloat16* orow = out + row * ldo + nb * kBN;
#pragma unroll 1
        for (int c = 0; c < kBN / 32; ++c) {
          uint32_t a[32];
          tmem_ld_32x32b_x32(taddr + c * 32, a);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float x0 = __uint_as_float(a[2 * j]), x1 = __uint_as_float(a[2 * j + 1]);
            if constexpr (kEpi == kEpiRelu) {
              x0 = fmaxf(x0, 0.0f);
              x1 = fmaxf(x1, 0.0f);
            }
            pk[j] = pack_bf16x2(x0, x1);
          }
          if (valid) {
#pragma unroll
            for (int v = 0; v < 4; ++v)
              st_global_v4(orow + c * 32 + v * 8, pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

int launch_grouped_gemm(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                        const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue,
                        void* out, const int32_t* slot_ready, int ready_from_slot, int epoch, cudaStream_t stream) {
  if (N % kBN != 0 || K % kBK != 0 || N <= 0 || K <= 0) return set_error(HM_EINVAL, "grouped_gemm: N %% 256 and K %% 64 must be 0");
  if (w_rows % N != 0) return set_error(HM_EINVAL, "grouped_gemm: weight rows must be a multiple of N");
  if (a_rows <= 0) return HM_OK;
  CUtensorMap ta, tb;
  int rc = make_tmap_2d_bf16(&ta, A, (uint64_t)a_rows, (uint64_t)K, kBM, kBK);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tb, W, (uint64_t)w_rows, (uint64_t)K, kBN, kBK);
  if (rc) return rc;
  const int ldo = (epilogue == kEpiSwiGLU) ? N / 2 : N;
  const int grid = num_sms();
  const int4* s4 = reinterpret_cast<const int4*>(segs);
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  switch (epilogue) {
    case kEpiStore:
      cudaFuncSetAttribute(grouped_gemm_kernel<kEpiStore>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
      grouped_gemm_kernel<kEpiStore><<<grid, kGemmThreads, kGemmSmem, stream>>>(
          ta, tb, s4, mtile_prefix, n_seg, o, N, K, ldo, slot_ready, ready_from_slot, epoch);
      break;
    case kEpiRelu:
      cudaFuncSetAttribute(grouped_gemm_kernel<kEpiRelu>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
      grouped_gemm_kernel<kEpiRelu><<<grid, kGemmThreads, kGemmSmem, stream>>>(
          ta, tb, s4, mtile_prefix, n_seg, o, N, K, ldo, slot_ready, ready_from_slot, epoch);
      break;
    case kEpiSwiGLU:
      cudaFuncSetAttribute(grouped_gemm_kernel<kEpiSwiGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
      grouped_gemm_kernel<kEpiSwiGLU><<<grid, kGemmThreads, kGemmSmem, stream>>>(
          ta, tb, s4, mtile_prefix, n_seg, o, N, K, ldo, slot_ready, ready_from_slot, epoch);
      break;
    default:
      return set_error(HM_EINVAL, "grouped_gemm: unknown epilogue");
  }
  return check_launch("grouped_gemm");
}

}  // namespace hm
