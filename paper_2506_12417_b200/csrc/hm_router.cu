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

#ifdef HM_ROUTER_STAMPS
// diagnostics build only (tools/router_stamps.py): per-tile %globaltimer stamps of the phases
__device__ unsigned long long g_rstamp[4096][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HM_RSTAMP(i) do { if (blockIdx.x < 4096) g_rstamp[blockIdx.x][i] = gtimer(); } while (0)
#else
#define HM_RSTAMP(i) do { } while (0)
#endif

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

// key[0..8) sorted descending (optimal 19-comparator network)
__device__ __forceinline__ void router_sort8(unsigned long long (&k)[8]) {
  ce_desc(k[0], k[2]); ce_desc(k[1], k[3]); ce_desc(k[4], k[6]); ce_desc(k[5], k[7]);
  ce_desc(k[0], k[4]); ce_desc(k[1], k[5]); ce_desc(k[2], k[6]); ce_desc(k[3], k[7]);
  ce_desc(k[0], k[1]); ce_desc(k[2], k[3]); ce_desc(k[4], k[5]); ce_desc(k[6], k[7]);
  ce_desc(k[2], k[4]); ce_desc(k[3], k[5]);
  ce_desc(k[1], k[4]); ce_desc(k[3], k[6]);
  ce_desc(k[1], k[2]); ce_desc(k[3], k[4]); ce_desc(k[5], k[6]);
}

// 32-bit compare-exchange / sorts for the truncated keys (2 instructions per comparator)
__device__ __forceinline__ void ce_u32(uint32_t& x, uint32_t& y) {
  const uint32_t hi = max(x, y), lo = min(x, y);
  x = hi;
  y = lo;
}
__device__ __forceinline__ void sort8_u32(uint32_t* k) {
  ce_u32(k[0], k[2]); ce_u32(k[1], k[3]); ce_u32(k[4], k[6]); ce_u32(k[5], k[7]);
  ce_u32(k[0], k[4]); ce_u32(k[1], k[5]); ce_u32(k[2], k[6]); ce_u32(k[3], k[7]);
  ce_u32(k[0], k[1]); ce_u32(k[2], k[3]); ce_u32(k[4], k[5]); ce_u32(k[6], k[7]);
  ce_u32(k[2], k[4]); ce_u32(k[3], k[5]);
  ce_u32(k[1], k[4]); ce_u32(k[3], k[6]);
  ce_u32(k[1], k[2]); ce_u32(k[3], k[4]); ce_u32(k[5], k[6]);
}
// A (sorted descending; na = the 9th largest of A's set, 0 if none) <- top-8 of A u B, na <- 9th
// largest of the union: the elementwise max of A and reversed B is a bitonic top-8, the
// elementwise min holds the bottom 8, whose maximum is the 9th
__device__ __forceinline__ void merge8_u32(uint32_t* A, uint32_t& na, const uint32_t* B, uint32_t nb) {
  uint32_t lo = max(na, nb);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t b = B[7 - i];
    lo = max(lo, min(A[i], b));
    A[i] = max(A[i], b);
  }
#pragma unroll
  for (int s2 = 4; s2 > 0; s2 >>= 1)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if ((i & s2) == 0) ce_u32(A[i], A[i + s2]);
  na = lo;
}
// key[0..8) <- the 8 largest of key[0..32), descending; ninth <- the 9th largest
__device__ __forceinline__ void top8_of_32_u32(uint32_t (&key)[32], uint32_t& ninth) {
#pragma unroll
  for (int g = 0; g < 32; g += 8) sort8_u32(key + g);
  uint32_t n0 = 0u, n2 = 0u;
  merge8_u32(key, n0, key + 8, 0u);
  merge8_u32(key + 16, n2, key + 24, 0u);
  merge8_u32(key, n0, key + 16, n2);
  ninth = n0;
}
// order-preserving uint32 (of a float, -0 folded into +0 as the float compare treats them) -> float
__device__ __forceinline__ float unord_u32(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;

// One 32-expert chunk of a row (2 < k <= 8 path): logits + bias, running (max, sum-exp) of the
// part, exact order-preserving keys (left in a[] for the shared-memory copy) and the truncated
// selection keys.  kGuard: the chunk extends past E (columns >= E are masked to -inf / key 0).
template <bool kGuard>
__device__ __forceinline__ void router_chunk(uint32_t (&a)[32], const float* __restrict__ sb, int nval,
                                             uint32_t kbase, float& pmx, float& psum, uint32_t (&key)[32]) {
  float cmx = -INFINITY;
  const float4* b4 = reinterpret_cast<const float4*>(sb);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 b = b4[i];
    const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int jj = 4 * i + h;
      float v = __fadd_rn(__uint_as_float(a[jj]), bb[h]);
      if (kGuard && jj >= nval) v = -INFINITY;
      a[jj] = __float_as_uint(v);
      cmx = fmaxf(cmx, v);
    }
  }
  const float nmx = fmaxf(pmx, cmx);  // finite: the chunk has at least one expert < E
  const float nb = -nmx * kLog2e;
  float cs = (pmx == -INFINITY) ? 0.0f : __fmul_rn(psum, ex2_ftz(__fmaf_rn(pmx, kLog2e, nb)));
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) cs = __fadd_rn(cs, ex2_ftz(__fmaf_rn(__uint_as_float(a[jj]), kLog2e, nb)));  // -inf -> 0
  pmx = nmx;
  psum = cs;
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) {
    uint32_t u = __float_as_uint(__fadd_rn(__uint_as_float(a[jj]), 0.0f));  // -0 -> +0
    u ^= static_cast<uint32_t>(static_cast<int32_t>(u) >> 31) | 0x80000000u;  // order-preserving
    a[jj] = u;
    key[jj] = (kGuard && jj >= nval) ? 0u : ((u & 0xFFFFFF00u) | (kbase - (uint32_t)jj));
  }
}

constexpr int kRBM = 128;
constexpr int kRBK = 64;
constexpr uint32_t kRPartBytes = 24 * 1024;  // epilogue partials (4 parts x 11 fields x 128 rows x 4 B)
constexpr int kRMaxStages = 8;
constexpr uint32_t kRA = kRBM * kRBK * 2;  // 16 KB
constexpr int kREpiWarps = 16;
constexpr int kRThreads = 64 + kREpiWarps * 32;
constexpr int kRKmax = 16;
constexpr size_t kREpiSmem = 2 * kRBM * kRKmax * sizeof(int) + 4 * 256 * sizeof(int) + 256 * sizeof(float);
constexpr size_t kRSmemMax = 227 * 1024;
// stages in flight: as many (A + Wg) k-blocks as fit (6 at E=128, 4 at E=256, 8 at E<=48)
inline int router_stages(int E_pad) {
  const size_t per = kRA + (size_t)E_pad * kRBK * 2;
  const size_t avail = kRSmemMax - 1024 - 256 - kREpiSmem;
  return (int)std::min<size_t>(kRMaxStages, avail / per);
}
}  // namespace

template <int KMAX>
__global__ void __maxnreg__(96)  // 18 warps: 5 on one SMSP x 96 x 32 <= 16K registers
    router_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                  const float* __restrict__ bias, int tokens_per_rank, int tiles_per_rank, int d, int E, int E_pad,
                  int k, int renorm, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                  int32_t* __restrict__ tile_hist, int32_t* __restrict__ lrank, int kRStages) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
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
  float* s_bias = reinterpret_cast<float*>(s_cnt + 4 * 256);  // [E_pad]: bias (0 without one)

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tile = blockIdx.x;
  const int rank = tile / tiles_per_rank;
  const int mt = tile - rank * tiles_per_rank;
  const int row0 = rank * tokens_per_rank + mt * kRBM;
  const int rows = min(kRBM, tokens_per_rank - mt * kRBM);
  const int KB = d / kRBK;
  const uint32_t b_bytes = (uint32_t)E_pad * kRBK * 2;
  if (threadIdx.x == 0) HM_RSTAMP(0);

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
      // (issued after the first ring's loads, which would otherwise queue behind the prefetches)
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < KB; ++kb) {
        if (kb == kRStages)
          for (int kp = kRStages; kp < KB; ++kp) tma_prefetch_l2_2d(&tmap_x, kp * kRBK, row0);
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
        if (kb == 0) HM_RSTAMP(1);
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
      HM_RSTAMP(7);
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
    // bias staged in shared memory: per-logit global loads behind per-element branches were
    // serialised round trips (the part phase's largest cost)
    for (int i = etid; i < E_pad; i += kREpiWarps * 32) s_bias[i] = (bias != nullptr && i < E) ? __ldg(bias + i) : 0.0f;
    named_bar_sync(2, kREpiWarps * 32);

    mbar_wait(&tfull[0], 0);
    if (etid == 0) HM_RSTAMP(2);
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
    float mx = -INFINITY, sum = 0.0f;
    if constexpr (KMAX == 4 || KMAX == 8) {
      // ---- 2 < k <= 8: selection on truncated 32-bit keys, made exact in the merge ----
      // (k <= 2 keeps the per-thread insertion below: measured faster for top-1/top-2)
      // key = (order-preserving value bits & ~0xFF) | (255 - expert): a comparator is 2 instructions
      // instead of 6 for the exact 64-bit (value, ~expert) key.  The truncation only matters for
      // distinct logits that agree in their upper 24 bits (within 2^-16 relative): the merge
      // re-sorts the selected experts by their exact keys and recomputes a row exactly when the
      // k-th and (k+1)-th truncated keys share a value bucket (so the selected SET could differ).
      // [128][32 * nchunk + 4] exact keys (every chunk stores all of its 32 columns)
      uint32_t* s_u = reinterpret_cast<uint32_t*>(smem + kRPartBytes);
      const int upitch = nchunk * 32 + 4;
      uint32_t lst[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) lst[j] = 0u;
      uint32_t ninth = 0u;
      float pmx = -INFINITY, psum = 0.0f;
      for (int c = part; c < nchunk; c += 4) {
        uint32_t a[32];
        tmem_ld_32x32b_x32(taddr + c * 32, a);
        tmem_ld_wait();
        uint32_t key[32];
        if (c * 32 + 32 <= E)
          router_chunk<false>(a, s_bias + c * 32, 32, 255u - (uint32_t)(c * 32), pmx, psum, key);
        else
          router_chunk<true>(a, s_bias + c * 32, E - c * 32, 255u - (uint32_t)(c * 32), pmx, psum, key);
        uint4* dst = reinterpret_cast<uint4*>(s_u + r * upitch + c * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = make_uint4(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]);
        uint32_t cn;
        top8_of_32_u32(key, cn);
        if (c == part) {
#pragma unroll
          for (int j = 0; j < 8; ++j) lst[j] = key[j];
          ninth = cn;
        } else {
          merge8_u32(lst, ninth, key, cn);
        }
      }
      // partials -> smem (aliases the drained pipeline stages): [part][field][row], fields
      // 0 max, 1 sum-exp, 2..9 sorted truncated keys, 10 the 9th key
      uint32_t* pu = reinterpret_cast<uint32_t*>(smem);
      {
        const int b = part * 11 * kRBM;
        pu[b + r] = __float_as_uint(pmx);
        pu[b + kRBM + r] = __float_as_uint(psum);
#pragma unroll
        for (int j = 0; j < 8; ++j) pu[b + (2 + j) * kRBM + r] = lst[j];
        pu[b + 10 * kRBM + r] = ninth;
      }
      named_bar_sync(2, kREpiWarps * 32);
      if (etid == 0) HM_RSTAMP(3);
      // ---- merge, outputs and ranks on all 16 warps: 4 adjacent lanes per row ----
      // (the partials are in shared memory, so rows no longer follow the TMEM lane quarters)
      {
        const int mr = etid >> 2;  // row of the tile
        const int sub = etid & 3;  // part list it loads / output slots it writes
        const bool mvalid = mr < rows;
        uint32_t A[8], na;
#pragma unroll
        for (int j = 0; j < 8; ++j) A[j] = pu[sub * 11 * kRBM + (2 + j) * kRBM + mr];
        na = pu[sub * 11 * kRBM + 10 * kRBM + mr];
        const float pm = __uint_as_float(pu[sub * 11 * kRBM + mr]);
        const float ps = __uint_as_float(pu[sub * 11 * kRBM + kRBM + mr]);
        // butterfly over the 4 lanes: every lane ends with the row's top-8 and 9th (merge8 is
        // symmetric in its operands) and the row max
        float m4 = pm;
#pragma unroll
        for (int sh = 1; sh <= 2; sh <<= 1) {
          uint32_t B[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) B[j] = __shfl_xor_sync(0xffffffffu, A[j], sh);
          const uint32_t nb = __shfl_xor_sync(0xffffffffu, na, sh);
          merge8_u32(A, na, B, nb);
          m4 = fmaxf(m4, __shfl_xor_sync(0xffffffffu, m4, sh));
        }
        mx = m4;
        // sum-exp: every lane rescales its part's partial, pairwise butterfly adds (commutative,
        // so all 4 lanes hold the bit-identical sum)
        float sm = (pm == -INFINITY) ? 0.0f : __fmul_rn(ps, __expf(__fsub_rn(pm, mx)));
#pragma unroll
        for (int sh = 1; sh <= 2; sh <<= 1) sm = __fadd_rn(sm, __shfl_xor_sync(0xffffffffu, sm, sh));
        sum = sm;
        // the k-th and (k+1)-th truncated keys
        uint32_t kth = 0u, nxt = na;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j == k - 1) kth = A[j];
          if (j == k) nxt = A[j];
        }
        const uint32_t* urow = s_u + mr * upitch;
        unsigned long long K[8];
        if (nxt == 0u || (kth >> 8) != (nxt >> 8)) {
          // every unselected expert is in a lower value bucket: the set is exact; exact keys
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            K[j] = 0ull;
            if (j < k) {
              const uint32_t id = 255u - (A[j] & 0xFFu);
              K[j] = (static_cast<unsigned long long>(urow[id]) << 32) | (0xFFFFFFFFu - id);
            }
          }
        } else {
          // ambiguous bucket at the boundary: exact top-k over the experts whose value bucket is at
          // least the k-th's (the selected higher buckets plus that bucket's members); the row's 4
          // lanes each scan a quarter of it, then two 64-bit top-8 butterfly merges
          const uint32_t bucket = kth >> 8;
#pragma unroll
          for (int j = 0; j < 8; ++j) K[j] = 0ull;
          const int q4 = (E + 15) / 16 * 4;  // quarter length, a multiple of 4
          const int e_lo = sub * q4, e_hi = min(E, e_lo + q4);
          for (int e4 = e_lo; e4 < e_hi; e4 += 4) {
            const uint4 u4 = *reinterpret_cast<const uint4*>(urow + e4);
            const uint32_t uu[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (e4 + i < e_hi && (uu[i] >> 8) >= bucket) {
                unsigned long long cv =
                    (static_cast<unsigned long long>(uu[i]) << 32) | (0xFFFFFFFFu - (uint32_t)(e4 + i));
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  if (cv > K[j]) {
                    const unsigned long long tk = K[j];
                    K[j] = cv;
                    cv = tk;
                  }
                }
              }
            }
          }
          // all 4 lanes of the row take this branch together (their condition is the row's)
#pragma unroll
          for (int sh = 1; sh <= 2; sh <<= 1) {
            unsigned long long O[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) O[j] = __shfl_xor_sync(0xFu << (lane & ~3), K[j], sh);
#pragma unroll
            for (int j = 0; j < 8; ++j) K[j] = K[j] > O[7 - j] ? K[j] : O[7 - j];
#pragma unroll
            for (int s2 = 4; s2 > 0; s2 >>= 1)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if ((j & s2) == 0) ce_desc(K[j], K[j + s2]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j >= k) K[j] = 0ull;
        }
        // lane sub owns selected entries j = sub, sub + 4: its exact slot is its rank among the k
        // exact keys (order: value desc, expert asc)
        float pw[2] = {0.0f, 0.0f};
        int slot[2] = {0, 0}, sid[2] = {-1, -1};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = sub + 4 * h;
          unsigned long long kj = 0ull;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (i == j) kj = K[i];
          int rk = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) rk += (K[i] > kj) ? 1 : 0;
          if (j < k) {
            slot[h] = rk;
            sid[h] = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(kj));
            pw[h] = __fdiv_rn(__expf(__fsub_rn(unord_u32(static_cast<uint32_t>(kj >> 32)), mx)), sum);
          }
        }
        if (renorm) {
          // sum of the k probabilities in slot order (fixed order; the 4 lanes exchange them)
          float ps_all = 0.0f;
#pragma unroll
          for (int sl = 0; sl < 8; ++sl) {
            float v = 0.0f;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (sid[h] >= 0 && slot[h] == sl) v = pw[h];
            // exactly one lane of the row holds slot sl: a max-free OR of the 4 lanes' values
            const uint32_t b = __float_as_uint(v);
            const uint32_t b1 = b | __shfl_xor_sync(0xffffffffu, b, 1);
            const uint32_t b2 = b1 | __shfl_xor_sync(0xffffffffu, b1, 2);
            if (sl < k) ps_all = __fadd_rn(ps_all, __uint_as_float(b2));
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (sid[h] >= 0) pw[h] = __fdiv_rn(pw[h], ps_all);
        }
        const int64_t tm = (int64_t)row0 + mr;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (sid[h] >= 0) {
            if (mvalid) {
              topk_idx[tm * k + slot[h]] = sid[h];
              topk_w[tm * k + slot[h]] = pw[h];
            }
            s_idx[mr * k + slot[h]] = mvalid ? sid[h] : -1;
          }
        }
      }
      // per-warp expert counts for the (token, slot)-order ranks: [16][E_pad] after s_u
      int* s_c16 = reinterpret_cast<int*>(smem + kRPartBytes + (size_t)kRBM * upitch * 4);
      for (int i = etid; i < kREpiWarps * E_pad; i += kREpiWarps * 32) s_c16[i] = 0;
      named_bar_sync(2, kREpiWarps * 32);
      if (etid == 0) HM_RSTAMP(4);
      // rank pass: warp ew walks the assignments of rows 8ew..8ew+7 in (token, slot) order
      const int abase = ew * 8 * k;
      int lr[2] = {0, 0}, le[2] = {-1, -1};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c * 32 < 8 * k) {
          const int a = c * 32 + lane;
          const int e = (a < 8 * k) ? s_idx[abase + a] : -1;
          const uint32_t mask = __match_any_sync(0xffffffffu, e);
          const int cnt0 = (e >= 0) ? s_c16[ew * E_pad + e] : 0;
          __syncwarp();
          if (e >= 0 && lane == 31 - __clz(mask)) s_c16[ew * E_pad + e] = cnt0 + __popc(mask);
          lr[c] = cnt0 + __popc(mask & lanemask_lt());
          le[c] = e;
          __syncwarp();
        }
      }
      named_bar_sync(2, kREpiWarps * 32);
      // exclusive prefix of the 16 warps' counts per expert; the tile histogram
      for (int e = etid; e < E_pad; e += kREpiWarps * 32) {
        int run = 0;
#pragma unroll
        for (int g = 0; g < kREpiWarps; ++g) {
          const int v = s_c16[g * E_pad + e];
          s_c16[g * E_pad + e] = run;
          run += v;
        }
        if (e < E) tile_hist[(int64_t)tile * E + e] = run;
      }
      named_bar_sync(2, kREpiWarps * 32);
      if (etid == 0) HM_RSTAMP(5);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int a = c * 32 + lane;
        if (c * 32 < 8 * k && a < 8 * k && le[c] >= 0)
          lrank[(int64_t)row0 * k + abase + a] = lr[c] + s_c16[ew * E_pad + le[c]];
      }
    } else {
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
          v = __fadd_rn(__uint_as_float(a[jj]), s_bias[e]);
        }
        a[jj] = __float_as_uint(v);
        mx = fmaxf(mx, v);
      }
      float cs = 0.0f;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        if (c * 32 + jj < E) cs = __fadd_rn(cs, ex2_ftz(__fmul_rn(__fsub_rn(__uint_as_float(a[jj]), mx), kLog2e)));
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
          v = __fadd_rn(__uint_as_float(a[jj]), s_bias[e]);
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
        if (c * 32 + jj < E) cs = __fadd_rn(cs, ex2_ftz(__fmul_rn(__fsub_rn(vals[jj], m), kLog2e)));
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
          v = __fadd_rn(__uint_as_float(a[jj]), s_bias[e]);
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
      float cs = (m_old == -INFINITY) ? 0.0f : __fmul_rn(lsum, ex2_ftz(__fmul_rn(__fsub_rn(m_old, m), kLog2e)));
#pragma unroll
      for (int jj = 0; jj < 32; ++jj)
        if (c * 32 + jj < E) cs = __fadd_rn(cs, ex2_ftz(__fmul_rn(__fsub_rn(vals[jj], m), kLog2e)));
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
    if (etid == 0) HM_RSTAMP(3);
    if (part == 0) {
    // merge: global max / sum-exp, and a 4-way merge of the sorted partial lists
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) mx = fmaxf(mx, pf[pp * nf * kRBM + r]);
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
      const float pm = pf[pp * nf * kRBM + r];
      if (pm != -INFINITY) sum = __fadd_rn(sum, __fmul_rn(pf[pp * nf * kRBM + kRBM + r], ex2_ftz(__fmul_rn(__fsub_rn(pm, mx), kLog2e))));
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
    }  // part == 0 (merge)
    if (part == 0) {
    float p[KMAX];
    float psum = 0.0f;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < k) {
        p[j] = __fdiv_rn(ex2_ftz(__fmul_rn(__fsub_rn(tv[j], mx), kLog2e)), sum);
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
    if (etid == 0) HM_RSTAMP(4);

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
    if (etid == 0) HM_RSTAMP(5);
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
    }  // k <= 2 or k > 8
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) HM_RSTAMP(6);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem_base);
  }
}

// ==========================================================================================
// Router v2: split-K over a cluster of C CTAs per 128-token tile.
//
// One 128-row tile per cluster; CTA c of the cluster multiplies its K slice (k-blocks
// [c*KB/C, (c+1)*KB/C)) into its own TMEM, then every CTA ships each row's partial logits to
// the row's owner (CTA r / (128/C)) through distributed shared memory; owners add the C
// partials in fixed order (so a token's logits never depend on the batch size) and run
// softmax + top-k on their 128/C rows, one thread per (row, 32-expert part); the per-tile
// histogram and the (token, slot)-order ranks combine the CTAs' counts through DSMEM too.
// At 16k tokens this spreads the tile's loads and its selection work over C SMs instead of
// one (grid 8x larger, several CTAs resident per SM); at small token counts (one EP rank's
// 2k tokens = 16 tiles) it is the difference between 16 busy SMs and 128.
// ==========================================================================================
constexpr int kR2EpiWarps = 8;
constexpr int kR2Threads = 64 + kR2EpiWarps * 32;

struct R2Layout {  // shared-memory carve-up, identical on host and device
  uint32_t region0;  // pipeline stages, later the partial-logit receive buffer
  uint32_t recv;     // [C][R][E_pad + 4] fp32 (inside region0; row pitch padded against bank conflicts)
  uint32_t bars;     // mbarriers + TMEM slot (256 B)
  uint32_t sidx;     // [RR][k] int
  uint32_t srank;    // [RR][k] int
  uint32_t scnt;     // [NG][E_pad] int
  uint32_t sccnt;    // [C][E_pad] int
  uint32_t total;
};

__host__ __device__ inline R2Layout r2_layout(int C, int E, int E_pad, int k, int stages) {
  const int R = 128 / C, RR = R < 32 ? 32 : R, NG = (R + 31) / 32;
  R2Layout L{};
  const uint32_t stage_bytes = (uint32_t)(kRA + (uint32_t)E_pad * kRBK * 2);
  L.recv = 0;
  const uint32_t need = (uint32_t)C * (E_pad + 4) * R * 4;
  const uint32_t st = stages * stage_bytes;
  L.region0 = ((need > st ? need : st) + 1023) / 1024 * 1024;
  L.bars = L.region0;
  L.sidx = L.bars + 256;
  L.srank = L.sidx + RR * k * 4;
  L.scnt = L.srank + RR * k * 4;
  L.sccnt = L.scnt + NG * E_pad * 4;
  L.total = L.sccnt + C * E_pad * 4;
  (void)E;
  return L;
}

template <int C>
__global__ void __launch_bounds__(kR2Threads)
    router_split_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                        const float* __restrict__ bias, int tokens_per_rank, int tiles_per_rank, int d, int E,
                        int E_pad, int k, int renorm, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                        int32_t* __restrict__ tile_hist, int32_t* __restrict__ lrank, int stages, uint32_t tmem_cols) {
  constexpr int R = 128 / C;
  constexpr int RR = R < 32 ? 32 : R;
  constexpr int NG = (R + 31) / 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const R2Layout L = r2_layout(C, E, E_pad, k, stages);
  const uint32_t stage_b = (uint32_t)E_pad * kRBK * 2;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + stages * kRA;
  float* recv = reinterpret_cast<float*>(smem + L.recv);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kRMaxStages;
  uint64_t* tfull = empty + kRMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  int* s_idx = reinterpret_cast<int*>(smem + L.sidx);
  int* s_rank = reinterpret_cast<int*>(smem + L.srank);
  int* s_cnt = reinterpret_cast<int*>(smem + L.scnt);
  int* s_ccnt = reinterpret_cast<int*>(smem + L.sccnt);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = cluster_ctarank();
  const int tile = blockIdx.x / C;
  const int rnk = tile / tiles_per_rank;
  const int mt = tile - rnk * tiles_per_rank;
  const int row0 = rnk * tokens_per_rank + mt * kRBM;
  const int rows = min(kRBM, tokens_per_rank - mt * kRBM);
  const int KB = d / kRBK;
  const int kb0 = (int)crank * KB / C, kb1 = ((int)crank + 1) * KB / C;

  if (warp == 0 && lane == 0) {
    for (int st = 0; st < stages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    mbar_init(&tfull[0], 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_w);
  }
  if (warp == 1) tmem_alloc_rt(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_x = l2_policy_evict_first();
      const uint64_t pol_w = l2_policy_evict_last();
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], kRA + stage_b);
        tma_load_2d(smem_a + st * kRA, &tmap_x, &full[st], kb * kRBK, row0, pol_x);
        tma_load_2d(smem_b + st * stage_b, &tmap_w, &full[st], kb * kRBK, 0, pol_w);
        if (++st == stages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(kRBM, (uint32_t)E_pad);
      int st = 0;
      uint32_t ph = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint64_t a0 = make_sdesc_sw128(smem_u32(smem_a + st * kRA));
        const uint64_t b0 = make_sdesc_sw128(smem_u32(smem_b + st * stage_b));
#pragma unroll
        for (int kk = 0; kk < kRBK / 16; ++kk)
          umma_bf16(tmem_base, a0 + (uint64_t)(kk * 2), b0 + (uint64_t)(kk * 2), idesc, (kb > kb0 || kk != 0));
        umma_commit(&empty[st]);
        if (++st == stages) {
          st = 0;
          ph ^= 1;
        }
      }
      umma_commit(&tfull[0]);
    }
  } else {
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
  }
  __syncwarp();
  // #1: every CTA's MMAs are complete, so every CTA's stage buffers may now be overwritten
  cluster_sync();

  const int ew = warp - 2;              // epilogue warp 0..7 (warps 0/1 join the later phases)
  const int etid = threadIdx.x - 64;    // 0..255 for epilogue threads
  if (ew >= 0) {
    // ship this CTA's partial logits: warp ew drains TMEM lane quarter (warp % 4) (hardware rule),
    // 32-column chunks ew/4, ew/4 + 2, ...; row r goes to CTA r / R as [src][row][e] (16-byte
    // remote stores)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t pitch = (uint32_t)E_pad + 4;
    const uint32_t dst = mapa_shared(recv, (uint32_t)(r / R)) + ((crank * R + (uint32_t)(r % R)) * pitch) * 4;
    const int nch = (E_pad + 31) / 32;
    for (int ch = ew >> 2; ch < nch; ch += 2) {
      uint32_t a[32];
      tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + ch * 32, a);
      tmem_ld_wait();
#pragma unroll
      for (int jj = 0; jj < 32; jj += 4)
        if (ch * 32 + jj < E_pad)
          asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + (ch * 32 + jj) * 4),
                       "r"(a[jj]), "r"(a[jj + 1]), "r"(a[jj + 2]), "r"(a[jj + 3])
                       : "memory");
    }
  }
  // #2: all partials delivered to their owners
  cluster_sync();

  if (ew >= 0) {
    // owner epilogue, lane-parallel: a row's experts are spread over LPR lanes (8 logits each);
    // every lane sorts its 8 packed (value, ~expert) keys, LPR-lane butterfly merges leave the
    // row's top-8 on every lane (ties: lowest expert id), then max / sum-exp by butterflies
    // (exact-commutative pairwise adds: every lane holds the bit-identical sum)
    const int lpr = E <= 128 ? 16 : 32;
    const int rpw = 32 / lpr;  // rows per warp and pass
    for (int rb = ew * rpw; rb < RR; rb += kR2EpiWarps * rpw) {
      const int rl = rb + lane / lpr;
      const int part = lane % lpr;
      const bool have = rl < R;
      const bool valid = have && (int)crank * R + rl < rows;
      float v[8];
      unsigned long long key[8];
      float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (have && part * 8 < E_pad) {
#pragma unroll
        for (int c = 0; c < C; ++c) {  // fixed order over the K slices
          const float4* src = reinterpret_cast<const float4*>(recv + ((uint32_t)c * R + rl) * (E_pad + 4) + part * 8);
          const float4 lo = src[0], hi = src[1];
          sum8[0] = __fadd_rn(sum8[0], lo.x); sum8[1] = __fadd_rn(sum8[1], lo.y);
          sum8[2] = __fadd_rn(sum8[2], lo.z); sum8[3] = __fadd_rn(sum8[3], lo.w);
          sum8[4] = __fadd_rn(sum8[4], hi.x); sum8[5] = __fadd_rn(sum8[5], hi.y);
          sum8[6] = __fadd_rn(sum8[6], hi.z); sum8[7] = __fadd_rn(sum8[7], hi.w);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int e = part * 8 + jj;
        float x = -INFINITY;
        if (have && e < E) {
          x = sum8[jj];
          if (bias != nullptr) x = __fadd_rn(x, __ldg(bias + e));
        }
        v[jj] = x;
        unsigned long long kv = (static_cast<unsigned long long>(0x007FFFFFu) << 32) | 0x80000000u;  // -inf
        if (have && e < E) {
          uint32_t u = __float_as_uint(__fadd_rn(x, 0.0f));  // -0 == +0 like the float compare
          u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
          kv = (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(e));
        }
        key[jj] = kv;
      }
      router_sort8(key);
      for (int sh = 1; sh < lpr; sh <<= 1) {
        unsigned long long o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __shfl_xor_sync(0xffffffffu, key[i], sh);
#pragma unroll
        for (int i = 0; i < 8; ++i) key[i] = key[i] > o[7 - i] ? key[i] : o[7 - i];
#pragma unroll
        for (int s2 = 4; s2 > 0; s2 >>= 1)
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if ((i & s2) == 0) ce_desc(key[i], key[i + s2]);
      }
      const uint32_t u0 = static_cast<uint32_t>(key[0] >> 32);
      const float mx = __uint_as_float((u0 & 0x80000000u) ? (u0 & 0x7FFFFFFFu) : ~u0);
      float ls = 0.0f;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (part * 8 + jj < E) ls = __fadd_rn(ls, expf(__fsub_rn(v[jj], mx)));
      for (int sh = 1; sh < lpr; sh <<= 1) ls = __fadd_rn(ls, __shfl_xor_sync(0xffffffffu, ls, sh));
      if (part == 0 && rl < RR) {
        if (!valid) {
          for (int j = 0; j < k; ++j) s_idx[rl * k + j] = -1;
        } else {
          const int64_t t = (int64_t)row0 + crank * R + rl;
          float pr[8];
          float psum = 0.0f;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < k) {
              const uint32_t u = static_cast<uint32_t>(key[j] >> 32);
              const float tv = __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
              pr[j] = __fdiv_rn(expf(__fsub_rn(tv, mx)), ls);
              psum = __fadd_rn(psum, pr[j]);
            }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < k) {
              const int id = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(key[j]));
              topk_idx[t * k + j] = id;
              topk_w[t * k + j] = renorm ? __fdiv_rn(pr[j], psum) : pr[j];
              s_idx[rl * k + j] = id;
            }
        }
      }
    }
    for (int i = etid; i < NG * E_pad; i += kR2EpiWarps * 32) s_cnt[i] = 0;
    named_bar_sync(2, kR2EpiWarps * 32);

    // rank pass: epilogue warp g walks row group g's assignments in (token, slot) order
    if (ew < NG) {
      const int g = ew;
      for (int c = 0; c < k; ++c) {
        const int a = g * 32 * k + c * 32 + lane;
        const int e = s_idx[a];
        const uint32_t mask = __match_any_sync(0xffffffffu, e);
        const int cnt0 = (e >= 0) ? s_cnt[g * E_pad + e] : 0;
        __syncwarp();
        const int leader = 31 - __clz(mask);
        if (e >= 0 && lane == leader) s_cnt[g * E_pad + e] = cnt0 + __popc(mask);
        s_rank[a] = cnt0 + __popc(mask & lanemask_lt());
        __syncwarp();
      }
    }
    named_bar_sync(2, kR2EpiWarps * 32);
    // this CTA's per-expert totals to every CTA of the cluster
    for (int e = etid; e < E_pad; e += kR2EpiWarps * 32) {
      int tot = 0;
      for (int g = 0; g < NG; ++g) tot += s_cnt[g * E_pad + e];
      for (int c = 0; c < C; ++c) st_cluster_s32(mapa_shared(s_ccnt + crank * E_pad + e, (uint32_t)c), tot);
    }
  }
  __syncwarp();
  // #3: all CTAs' totals in place
  cluster_sync();
  if (ew >= 0) {
    for (int rl = etid; rl < R; rl += kR2EpiWarps * 32) {
      if ((int)crank * R + rl >= rows) continue;
      const int64_t t = (int64_t)row0 + crank * R + rl;
      const int g = rl / 32;
      for (int j = 0; j < k; ++j) {
        const int e = s_idx[rl * k + j];
        int off = 0;
        for (int gg = 0; gg < g; ++gg) off += s_cnt[gg * E_pad + e];
        for (int c = 0; c < (int)crank; ++c) off += s_ccnt[c * E_pad + e];
        lrank[t * k + j] = s_rank[rl * k + j] + off;
      }
    }
    for (int e = (int)crank + C * etid; e < E; e += C * kR2EpiWarps * 32) {
      int tot = 0;
      for (int c = 0; c < C; ++c) tot += s_ccnt[c * E_pad + e];
      tile_hist[(int64_t)tile * E + e] = tot;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_rt(tmem_base, tmem_cols);
  }
}

// HM_ROUTER_V2=1: the split-K cluster kernel above (opt-in experiment, profiles/r2_experiments.txt:
// correct and bit-exact on the router tests, but slower than the one-CTA-per-tile kernel at
// 16k tokens - 49-113 us vs 37-43 us cold for C = 2..8 - because launching thousands of
// cluster CTAs and three cluster barriers per tile cost more than the split saves; it wins
// only at small token counts (2k tokens: 27-31 us vs 39 us) and a token's logits must not
// depend on the batch size, so the variant cannot be chosen per call)
static bool use_router_v1() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HM_ROUTER_V2");
    v = (e != nullptr && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

template <int C>
static int launch_router_split(const CUtensorMap& tx, const CUtensorMap& tw, const float* bias, int tokens_per_rank,
                               int tiles_per_rank, int n_tiles, int d, int E, int E_pad, int k, int renormalize,
                               int32_t* topk_idx, float* topk_w, int32_t* tile_hist, int32_t* lrank,
                               cudaStream_t stream) {
  const int KB = d / kRBK;
  const int kbc = (KB + C - 1) / C;
  int stages = kbc < 2 ? kbc : 2;
  if (const char* e = getenv("HM_ROUTER_STAGES")) stages = std::max(1, std::min(kRMaxStages, std::min(kbc, atoi(e))));
  const R2Layout L = r2_layout(C, E, E_pad, k, stages);
  const size_t smem = 1024 + L.total;
  uint32_t cols = 32;
  while ((int)cols < E_pad) cols <<= 1;
  cudaFuncSetAttribute(router_split_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_tiles * C));
  cfg.blockDim = dim3(kR2Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, router_split_kernel<C>, tx, tw, bias, tokens_per_rank,
                                           tiles_per_rank, d, E, E_pad, k, renormalize, topk_idx, topk_w, tile_hist,
                                           lrank, stages, cols);
  if (e != cudaSuccess) return set_error(HM_ECUDA, "router (split) launch: %s", cudaGetErrorString(e));
  return check_launch("router_topk");
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
  if (!use_router_v1() && k <= 8) {
    // cluster size by the model width only (never by the batch size: a token's logits must not
    // depend on how many other tokens are routed with it): up to 8 k-slices of >= 1 k-block
    const int KB = d / kRBK;
    int C = KB >= 8 ? 8 : (KB >= 4 ? 4 : (KB >= 2 ? 2 : 1));
    if (const char* ce = getenv("HM_ROUTER_C")) C = std::max(1, std::min(C, atoi(ce)));
#define HM_R2(CC)                                                                                               \
  return launch_router_split<CC>(tx, tw, bias, tokens_per_rank, tiles_per_rank, grid, d, E, E_pad, k, renormalize, \
                                 topk_idx, topk_w, tile_hist, lrank, stream)
    switch (C) {
      case 1: HM_R2(1);
      case 2: HM_R2(2);
      case 4: HM_R2(4);
      default: HM_R2(8);
    }
#undef HM_R2
  }
  const int stages = router_stages(E_pad);
  // the 2 < k <= 8 epilogue reuses the drained ring for its partials and exact keys
  if ((size_t)stages * (kRA + (size_t)E_pad * kRBK * 2) <
      kRPartBytes + (size_t)kRBM * ((E + 31) / 32 * 32 + 4) * 4 + (size_t)kREpiWarps * E_pad * 4)
    return set_error(HM_EINVAL, "router: pipeline ring too small for the epilogue scratch (E_pad %d)", E_pad);
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

#ifdef HM_ROUTER_STAMPS
namespace hm {
__global__ void debug_stamp_kernel(int slot) { g_rstamp[4095][slot] = gtimer(); }
}  // namespace hm
// one-thread kernel writing %globaltimer into g_rstamp[4095][slot] (launch-gap measurements)
extern "C" __attribute__((visibility("default"))) int hm_debug_stamp(int slot, void* stream) {
  hm::debug_stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(slot);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int hm_debug_router_stamps(void* out, int n_tiles) {
  return cudaMemcpyFromSymbol(out, hm::g_rstamp, (size_t)n_tiles * 8 * sizeof(unsigned long long)) == cudaSuccess ? 0 : 1;
}
#endif
