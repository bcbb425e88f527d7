// K1 + K2: router (gate GEMM + softmax + top-k) fused with the per-tile expert
// histogram and the deterministic (token, slot)-order rank pass.
//
// Replaces Alg.1 step 1 whose reference stand-in is
// workload.sample_routing (workload.py:167-180), and builds the per-GPU
// token->expert histogram that becomes RoutingMatrix.counts[g] (core.py:89-96),
// i.e. the 4 KB metadata exchanged in step 2.
//
// One CTA per 128-token tile.  Logits [128, E_pad] accumulate in TMEM via
// tcgen05.mma (A = x tile via TMA, B = Wg via TMA); the 4 epilogue warps own one
// token row each (TMEM lane == row) and run softmax + top-k in registers.
// Top-k is taken over the fp32 logits, ties to the lowest expert id; weights are
// the softmax probabilities of the winners (optionally renormalised over k).
// The rank pass uses __match_any_sync over 32-assignment chunks in (token, slot)
// order so lrank is deterministic (no atomics), which is what makes the
// dispatch bit-reproducible.
#include <algorithm>

#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

namespace {
// descending compare-exchange on packed keys
__device__ __forceinline__ void ce_desc(unsigned long long& x, unsigned long long& y) {
  const unsigned long long hi = x > y ? x : y;
  const unsigned long long lo = x > y ? y : x;
  x = hi;
  y = lo;
}

// key[0..8) <- the 8 largest of key[0..32), descending
__device__ __forceinline__ void router_top8_of_32(unsigned long long (&key)[32]) {
  // optimal 19-comparator network for 8 elements, applied to the four groups of 8
#pragma unroll
  for (int g = 0; g < 32; g += 8) {
    unsigned long long* k = key + g;
    ce_desc(k[0], k[2]); ce_desc(k[1], k[3]); ce_desc(k[4], k[6]); ce_desc(k[5], k[7]);
    ce_desc(k[0], k[4]); ce_desc(k[1], k[5]); ce_desc(k[2], k[6]); ce_desc(k[3], k[7]);
    ce_desc(k[0], k[1]); ce_desc(k[2], k[3]); ce_desc(k[4], k[5]); ce_desc(k[6], k[7]);
    ce_desc(k[2], k[4]); ce_desc(k[3], k[5]);
    ce_desc(k[1], k[4]); ce_desc(k[3], k[6]);
    ce_desc(k[1], k[2]); ce_desc(k[3], k[4]); ce_desc(k[5], k[6]);
  }
  // top-8 of two sorted runs: elementwise max against the reversed run is bitonic and holds
  // the 8 largest; three half-cleaner stages sort it
#pragma unroll
  for (int step = 8; step < 32; step *= 2) {
#pragma unroll
    for (int g = 0; g < 32; g += 2 * step) {
      unsigned long long* A = key + g;
      const unsigned long long* B = key + g + step;
#pragma unroll
      for (int i = 0; i < 8; ++i) A[i] = A[i] > B[7 - i] ? A[i] : B[7 - i];
#pragma unroll
      for (int s2 = 4; s2 > 0; s2 >>= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if ((i & s2) == 0) ce_desc(A[i], A[i + s2]);
    }
  }
}

constexpr int kRBM = 128;
constexpr int kRBK = 64;
constexpr int kRMaxStages = 8;
constexpr uint32_t kRA = kRBM * kRBK * 2;  // 16 KB
constexpr int kREpiWarps = 16;
constexpr int kRThreads = 64 + kREpiWarps * 32;
constexpr int kRKmax = 16;
constexpr size_t kREpiSmem = 2 * kRBM * kRKmax * sizeof(int) + 4 * 256 * sizeof(int);
constexpr size_t kRSmemMax = 227 * 1024;
// stages in flight: as many (A + Wg) k-blocks as fit (6 at E=128, 4 at E=256, 8 at E<=48)
inline int router_stages(int E_pad) {
  const size_t per = kRA + (size_t)E_pad * kRBK * 2;
  const size_t avail = kRSmemMax - 1024 - 256 - kREpiSmem;
  return (int)std::min<size_t>(kRMaxStages, avail / per);
}
}  // namespace

template <int KMAX>
__global__ void __maxnreg__(104)
    router_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                  const float* __restrict__ bias, int tokens_per_rank, int tiles_per_rank, int d, int E, int E_pad,
                  int k, int renorm, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                  int32_t* __restrict__ tile_hist, int32_t* __restrict__ lrank, int kRStages) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t kRBmax = (uint32_t)E_pad * kRBK * 2;  // B stage stride (multiple of 2 KB)
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kRStages * kRA;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_b + kRStages * kRBmax);
  uint64_t* empty = full + kRMaxStages;
  uint64_t* tfull = empty + kRMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  int* s_idx = reinterpret_cast<int*>(smem_b + kRStages * kRBmax + 256);
  int* s_rank = s_idx + kRBM * kRKmax;
  int* s_cnt = s_rank + kRBM * kRKmax;  // [4][E_pad]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tile = blockIdx.x;
  const int rank = tile / tiles_per_rank;
  const int mt = tile - rank * tiles_per_rank;
  const int row0 = rank * tokens_per_rank + mt * kRBM;
  const int rows = min(kRBM, tokens_per_rank - mt * kRBM);
  const int KB = d / kRBK;
  const uint32_t b_bytes = (uint32_t)E_pad * kRBK * 2;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kRStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_w);
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_x = l2_policy_evict_first();
      const uint64_t pol_w = l2_policy_evict_last();
      // the whole x tile (128 rows x d) is requested from HBM up front; the staged
      // TMA loads below then hit L2 instead of exposing DRAM latency per stage
      // fixed K order for every tile: a token's logits do not depend on its position in
      // the batch (chunked / micro-batched forwards route identically)
      for (int kb = kRStages; kb < KB; ++kb) tma_prefetch_l2_2d(&tmap_x, kb * kRBK, row0);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], kRA + b_bytes);
        tma_load_2d(smem_a + stage * kRA, &tmap_x, &full[stage], kb * kRBK, row0, pol_x);
        tma_load_2d(smem_b + stage * kRBmax, &tmap_w, &full[stage], kb * kRBK, 0, pol_w);
        if (++stage == kRStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(kRBM, (uint32_t)E_pad);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t a0 = make_sdesc_sw128(smem_u32(smem_a + stage * kRA));
        const uint64_t b0 = make_sdesc_sw128(smem_u32(smem_b + stage * kRBmax));
#pragma unroll
        for (int kk = 0; kk < kRBK / 16; ++kk)
          umma_bf16(tmem_base, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
        umma_commit(&empty[stage]);
        if (++stage == kRStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(&tfull[0]);
    }
  } else {
    // ===== epilogue: softmax + top-k + histogram/rank =====
    // 16 warps: 4 per TMEM lane quarter (hardware: warp id % 4); "part" p of a quarter scans
    // the 32-expert chunks p, p+4, ... of its 32 token rows, then part 0 merges the 4 partial
    // (top-k, max, sum-exp) results and runs the rank pass.
    const int ew = warp - 2;           // 0..15
    const int q = warp & 3;            // lane quarter
    const int part = ew >> 2;          // 0..3
    const int etid = threadIdx.x - 64; // 0..511
    const int r = q * 32 + lane;
    const bool valid = r < rows;
    const int64_t t = (int64_t)row0 + r;
    for (int i = etid; i < 4 * E_pad; i += kREpiWarps * 32) s_cnt[i] = 0;

    mbar_wait(&tfull[0], 0);
    tc_fence_after();
    const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16);

    float tv[KMAX];
    int ti[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      tv[j] = -INFINITY;
      ti[j] = 0x7fffffff;
    }
    const int nchunk = (E + 31) / 32;
    float vals[32];
    float lsum = 0.0f;
    // single pass per chunk: logits stay in registers for the partial sum-exp
    if (KMAX == 8 && part < nchunk) {
      // top-8 of this part's 32 logits as a sorting network over packed 64-bit keys
      // (order-preserving value bits << 32 | ~expert, so equal logits keep the lowest expert
      // first, as the insertion below does): four 19-comparator sorts of 8 and three
      // bitonic top-8 merges - 136 independent compare-exchanges instead of 256 dependent
      // insertion steps
      const int c = part;
      uint32_t a[32];
      tmem_ld_32x32b_x32(taddr + c * 32, a);
      tmem_ld_wait();
      // logits (bias added) in place, then max and partial sum-exp first so only the keys stay
      // live through the network
      float mx = -INFINITY;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int e = c * 32 + jj;
        float v = -INFINITY;
        if (e < E) {
          v = __uint_as_float(a[jj]);
          if (bias != nullptr) v = __fadd_rn(v, __ldg(bias + e));
        }
        a[jj] = __float_as_uint(v);
        mx = fmaxf(mx, v);
      }
      float cs = 0.0f;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        if (c * 32 + jj < E) cs = __fadd_rn(cs, expf(__fsub_rn(__uint_as_float(a[jj]), mx)));
      lsum = cs;
      unsigned long long key[32];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int e = c * 32 + jj;
        unsigned long long kv = (static_cast<unsigned long long>(0x007FFFFFu) << 32) | 0x80000000u;  // -inf, id INT_MAX
        if (e < E) {
          uint32_t u = __float_as_uint(__fadd_rn(__uint_as_float(a[jj]), 0.0f));  // -0 == +0 like the float compare
          u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
          kv = (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(e));
        }
        key[jj] = kv;
      }
      router_top8_of_32(key);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t u = static_cast<uint32_t>(key[j] >> 32);
        tv[j] = __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
        ti[j] = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(key[j]));
      }
    } else if (part < nchunk) {
      const int c = part;
      uint32_t a[32];
      tmem_ld_32x32b_x32(taddr + c * 32, a);
      tmem_ld_wait();
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int e = c * 32 + jj;
        float v = -INFINITY;
        if (e < E) {
          v = __uint_as_float(a[jj]);
          if (bias != nullptr) v = __fadd_rn(v, __ldg(bias + e));
          float cv = v;
          int ci = e;
          bool ins = false;
#pragma unroll
          for (int j = 0; j < KMAX; ++j) {
            if (j < k && (ins || cv > tv[j])) {
              const float tf = tv[j];
              const int tix = ti[j];
              tv[j] = cv;
              ti[j] = ci;
              cv = tf;
              ci = tix;
              ins = true;
            }
          }
        }
        vals[jj] = v;
      }
      // running partial sum of exp(v - m) with m = this part's running max (tv[0])
      const float m = tv[0];
      float cs = 0.0f;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        if (c * 32 + jj < E) cs = __fadd_rn(cs, expf(__fsub_rn(vals[jj], m)));
      lsum = cs;
    }
    for (int c = part + 4; c < nchunk; c += 4) {
      // second chunk of this part (E > 128): rescale the running sum to the new max
      uint32_t a[32];
      tmem_ld_32x32b_x32(taddr + c * 32, a);
      tmem_ld_wait();
      const float m_old = tv[0];
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int e = c * 32 + jj;
        float v = -INFINITY;
        if (e < E) {
          v = __uint_as_float(a[jj]);
          if (bias != nullptr) v = __fadd_rn(v, __ldg(bias + e));
          float cv = v;
          int ci = e;
          bool ins = false;
#pragma unroll
          for (int j = 0; j < KMAX; ++j) {
            if (j < k && (ins || cv > tv[j])) {
              const float tf = tv[j];
              const int tix = ti[j];
              tv[j] = cv;
              ti[j] = ci;
              cv = tf;
              ci = tix;
              ins = true;
            }
          }
        }
        vals[jj] = v;
      }
      const float m = tv[0];
      float cs = (m_old == -INFINITY) ? 0.0f : __fmul_rn(lsum, expf(__fsub_rn(m_old, m)));
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        if (c * 32 + jj < E) cs = __fadd_rn(cs, expf(__fsub_rn(vals[jj], m)));
      lsum = cs;
    }
    // partials -> smem (aliases the drained pipeline stages): [part][field][row]
    float* pf = reinterpret_cast<float*>(smem);
    int* pi = reinterpret_cast<int*>(smem);
    const int nf = 2 + 2 * KMAX;
    {
      const int b = part * nf * kRBM;
      pf[b + 0 * kRBM + r] = tv[0];
      pf[b + 1 * kRBM + r] = lsum;
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        pf[b + (2 + j) * kRBM + r] = tv[j];
        pi[b + (2 + KMAX + j) * kRBM + r] = ti[j];
      }
    }
    named_bar_sync(2, kREpiWarps * 32);
    if (part == 0) {
    // merge: global max / sum-exp, and a 4-way merge of the sorted partial lists
    float mx = -INFINITY;
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) mx = fmaxf(mx, pf[pp * nf * kRBM + r]);
    float sum = 0.0f;
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
      const float pm = pf[pp * nf * kRBM + r];
      if (pm != -INFINITY) sum = __fadd_rn(sum, __fmul_rn(pf[pp * nf * kRBM + kRBM + r], expf(__fsub_rn(pm, mx))));
    }
    {
      int head[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < k) {
          float bv = -INFINITY;
          int bi = 0x7fffffff, bp = 0;
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {
            if (head[pp] < k) {
              const float v = pf[pp * nf * kRBM + (2 + head[pp]) * kRBM + r];
              const int id = pi[pp * nf * kRBM + (2 + KMAX + head[pp]) * kRBM + r];
              if (v > bv || (v == bv && id < bi)) {
                bv = v;
                bi = id;
                bp = pp;
              }
            }
          }
          tv[j] = bv;
          ti[j] = bi;
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) head[pp] += (pp == bp);
        }
      }
    }
    float p[KMAX];
    float psum = 0.0f;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < k) {
        p[j] = __fdiv_rn(expf(__fsub_rn(tv[j], mx)), sum);
        psum = __fadd_rn(psum, p[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < k) {
        const float w = renorm ? __fdiv_rn(p[j], psum) : p[j];
        if (valid) {
          topk_idx[t * k + j] = ti[j];
          topk_w[t * k + j] = w;
        }
        s_idx[r * k + j] = valid ? ti[j] : -1;
      }
    }
    named_bar_sync(1, 128);

    // rank pass: warp q walks its 32 rows' assignments in (token, slot) order
    const int base_a = q * 32 * k;
    for (int c = 0; c < k; ++c) {
      const int a = base_a + c * 32 + lane;
      const int e = s_idx[a];
      const uint32_t mask = __match_any_sync(0xffffffffu, e);
      const int cnt0 = (e >= 0) ? s_cnt[q * E_pad + e] : 0;
      __syncwarp();
      const int leader = 31 - __clz(mask);
      if (e >= 0 && lane == leader) s_cnt[q * E_pad + e] = cnt0 + __popc(mask);
      s_rank[a] = cnt0 + __popc(mask & lanemask_lt());
      __syncwarp();
    }
    named_bar_sync(1, 128);
    if (valid) {
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < k) {
          const int e = ti[j];
          int off = 0;
          for (int qq = 0; qq < q; ++qq) off += s_cnt[qq * E_pad + e];
          lrank[t * k + j] = s_rank[r * k + j] + off;
        }
      }
    }
    for (int e = etid; e < E; e += 128)
      tile_hist[(int64_t)tile * E + e] =
          s_cnt[e] + s_cnt[E_pad + e] + s_cnt[2 * E_pad + e] + s_cnt[3 * E_pad + e];
    }  // part == 0
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem_base);
  }
}

int launch_router(const void* x, const void* wg, const float* bias, int n_ranks, int tokens_per_rank, int d, int E,
                  int k, int renormalize, int32_t* topk_idx, float* topk_w, int32_t* tile_hist, int32_t* lrank,
                  cudaStream_t stream) {
  if (n_ranks < 1 || tokens_per_rank < 0 || d <= 0 || d % 64 != 0)
    return set_error(HM_EINVAL, "router: need n_ranks >= 1 and d %% 64 == 0");
  if (E < 1 || E > 256 || k < 1 || k > kRKmax || k > E)
    return set_error(HM_EINVAL, "router: need 1 <= k <= min(E, 16) and E <= 256");
  if (tokens_per_rank == 0) return HM_OK;
  const int E_pad = (E + 15) / 16 * 16;
  const int tiles_per_rank = (tokens_per_rank + kRBM - 1) / kRBM;
  const int64_t T = (int64_t)n_ranks * tokens_per_rank;
  CUtensorMap tx, tw;
  int rc = make_tmap_2d_bf16(&tx, x, (uint64_t)T, (uint64_t)d, kRBM, kRBK);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tw, wg, (uint64_t)E_pad, (uint64_t)d, (uint32_t)E_pad, kRBK);
  if (rc) return rc;
  const int grid = n_ranks * tiles_per_rank;
  const int stages = router_stages(E_pad);
  const size_t smem = 1024 + (size_t)stages * (kRA + (size_t)E_pad * kRBK * 2) + 256 + kREpiSmem;
#define HM_LAUNCH_ROUTER(KM)                                                                                 \
  do {                                                                                                       \
    cudaFuncSetAttribute(router_kernel<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    router_kernel<KM><<<grid, kRThreads, smem, stream>>>(tx, tw, bias, tokens_per_rank, tiles_per_rank, d,   \
                                                         E, E_pad, k, renormalize, topk_idx, topk_w,         \
                                                         tile_hist, lrank, stages);                          \
  } while (0)
  if (k == 1) HM_LAUNCH_ROUTER(1);
  else if (k == 2) HM_LAUNCH_ROUTER(2);
  else if (k <= 4) HM_LAUNCH_ROUTER(4);
  else if (k <= 8) HM_LAUNCH_ROUTER(8);
  else HM_LAUNCH_ROUTER(16);
#undef HM_LAUNCH_ROUTER
  return check_launch("router_topk");
}

}  // namespace hm
