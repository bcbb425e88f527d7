// K5: grouped expert GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces the expert-compute phase the reference only models
// (moesim/engine.py:128-132 CostModel.expert_flops, engine.py:354-359 per-GPU
// execution; Alg.1 step 5).  Persistent CTAs walk a device-resident
// tile list built by hm_dispatch_layout (no host sync):
//
//   segment s = {row_start, nrows, wslot, expert}: rows [row_start, row_start+nrows)
//   of the token buffer A are multiplied by weight slot `wslot` (W[wslot] is
//   [N, K] K-major, i.e. nn.Linear layout).  Segments come in HarMoEny plan order
//   (engine.py:233-234: residents first, then fetched experts) so async weight fetches
//   (K6) get the longest possible compute shadow.
//
// Two kernels share the epilogue design:
// * grouped_gemm_2cta_kernel (default): CTA pairs (cluster of 2, tcgen05.mma.cta_group::2)
//   on 256 x 256 pair tiles; a segment's odd 128-row tail runs as an M=128 "half" tile;
//   the tile walk is m-major (or grouped by 16 m-tiles for experts whose weights do not fit
//   L2); A comes by TMA or, for the fused scatter, from cp.async loader warps that gather
//   token rows of x directly.  Described in detail above the kernel.
// * grouped_gemm_kernel (HM_GEMM_1CTA=1): one CTA per SM, 128 x 256 tiles, 4-stage ring.
//
// Epilogue: epilogue warp w owns TMEM lane quarter w%4 (32 rows) and one half of the
// tile's columns.  Each thread converts its row (TMEM -> regs -> bf16) into a padded
// per-warp smem staging tile, then the warp writes whole 64-byte row segments (8 rows per
// instruction), optionally scattered through row_map (the FFN2 output goes token-major
// so the combine streams contiguously).
//   kEpiStore (bf16 out), kEpiRelu (Switch FFN1), kEpiSwiGLU (W13 is block-
//   interleaved: within each 256-row block, rows [0,128) are gate rows and
//   [128,256) the matching up rows -> 128 bf16 outputs per tile).
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
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 64 + kEpiWarps * 32;
constexpr int kMaxSmemSegs = 512;                 // segment table staged in smem (10 KB) when it fits
constexpr int kStgCols = 32;                      // bf16 output columns per staging pass
constexpr int kStgPitch = kStgCols * 2 + 16;      // 80 B: conflict-free 16-byte row writes
constexpr int kStgBytes = 32 * kStgPitch;         // per epilogue warp
constexpr size_t kGemmSmem =
    1024 + kStages * (kABytes + kBBytes) + 256 + kMaxSmemSegs * 20 + 16 + kEpiWarps * kStgBytes;

// Persistent tile walk.  Tile t (increasing per CTA) -> segment via a monotone
// cursor (amortised O(1), no dependent global-memory search per tile).
struct TileCursor {
  const int4* segs;
  const int* mp;
  int NB;
  int s = 0;
  __device__ __forceinline__ void seek(int t, int4& seg, int& m, int& nb) {
    while (mp[s + 1] * NB <= t) ++s;
    seg = segs[s];
    const int ms = mp[s + 1] - mp[s];
    const int local = t - mp[s] * NB;
    nb = local / ms;
    m = local - nb * ms;
  }
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Convert 32 fp32 accumulator columns of this thread's row to bf16 and store them
// (64 B) into the warp's staging row.
template <int kEpi>
__device__ __forceinline__ void stage_row(uint32_t srow, const uint32_t (&a)[32], const uint32_t (&u)[32]) {
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = v * 8 + j * 2;
      float x0 = __uint_as_float(a[c]), x1 = __uint_as_float(a[c + 1]);
      if constexpr (kEpi == kEpiRelu) {
        x0 = fmaxf(x0, 0.0f);
        x1 = fmaxf(x1, 0.0f);
      } else if constexpr (kEpi == kEpiSwiGLU) {
        const float u0 = __uint_as_float(u[c]), u1 = __uint_as_float(u[c + 1]);
        x0 = x0 / (1.0f + __expf(-x0)) * u0;
        x1 = x1 / (1.0f + __expf(-x1)) * u1;
      }
      pk[j] = pack_bf16x2(x0, x1);
    }
    st_shared_v4(srow + v * 16, pk[0], pk[1], pk[2], pk[3]);
  }
}

template <int kEpi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const int4* __restrict__ segs_g, const int* __restrict__ mprefix_g,
                        const int* __restrict__ n_seg_ptr, __nv_bfloat16* __restrict__ out, int N, int K, int ldo,
                        const int* __restrict__ row_map, const int* __restrict__ a_gather, int a_gather_div,
                        int a_gather_rows, const int* __restrict__ slot_ready, int ready_from_slot, int epoch) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_b + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int4* s_segs = reinterpret_cast<int4*>(smem_b + kStages * kBBytes + 256);
  int* s_mp = reinterpret_cast<int*>(s_segs + kMaxSmemSegs);
  uint8_t* s_stage = reinterpret_cast<uint8_t*>(s_mp + kMaxSmemSegs + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_seg = *n_seg_ptr;
  const bool seg_in_smem = n_seg <= kMaxSmemSegs;
  if (seg_in_smem) {
    for (int i = threadIdx.x; i < n_seg; i += blockDim.x) s_segs[i] = segs_g[i];
    for (int i = threadIdx.x; i <= n_seg; i += blockDim.x) s_mp[i] = mprefix_g[i];
  }

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);
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

  const int NB = N / kBN;
  const int4* segs = seg_in_smem ? s_segs : segs_g;
  const int* mp = seg_in_smem ? s_mp : mprefix_g;
  const int total = n_seg > 0 ? mp[n_seg] * NB : 0;
  const int KB = K / kBK;

  if (warp == 0) {
    // ===== TMA producer (one lane; the whole warp when A rows are gathered) =====
    const uint64_t pol_a = l2_policy_evict_normal();
    const uint64_t pol_b = l2_policy_evict_last();
    const bool gather = a_gather != nullptr;
    TileCursor cur{segs, mp, NB};
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int4 seg;
      int m, nb;
      cur.seek(t, seg, m, nb);
      const int row0 = seg.x + m * kBM;
      const int brow = seg.z * N + nb * kBN;
      int gr[4];
      if (gather) {
        // lane l gathers tile rows 4l..4l+3: A row = a_gather[buffer row] / div (the token);
        // rows past the segment repeat a valid row (their results are never stored)
        const int valid = min(kBM, seg.y - m * kBM);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int rr = min(lane * 4 + j, valid - 1);
          gr[j] = min(__ldg(a_gather + row0 + rr) / a_gather_div, a_gather_rows - 1);
        }
      }
      if (lane == 0 && slot_ready != nullptr && seg.z >= ready_from_slot) {
        // K6: fetched expert weights land asynchronously; wait for this expert's epoch
        long long spins = 0;  // watchdog, as in the 2-CTA kernel
        while (ld_acquire_gpu(slot_ready + seg.w) < epoch) {
          __nanosleep(128);
          if (++spins > (1ll << 26)) __trap();
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      for (int kb = 0; kb < KB; ++kb) {
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kABytes + kBBytes);
          if (!gather) tma_load_2d(smem_a + stage * kABytes, &tmap_a, &full[stage], kb * kBK, row0, pol_a);
          tma_load_2d(smem_b + stage * kBBytes, &tmap_b, &full[stage], kb * kBK, brow, pol_b);
        }
        if (gather) {
          __syncwarp();
          tma_gather4(smem_a + stage * kABytes + lane * 512, &tmap_a, &full[stage], kb * kBK, gr[0], gr[1], gr[2],
                      gr[3], pol_a);
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
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
    // ===== epilogue: warps 2..9 =====
    const int ew = warp - 2;             // 0..7
    const int q = warp & 3;              // TMEM lane quarter (hardware: warp id % 4)
    const int half = ew >> 2;            // which half of the tile's output columns
    constexpr int kOutCols = (kEpi == kEpiSwiGLU) ? kBN / 2 : kBN;  // bf16 outputs per tile row
    constexpr int kHalfCols = kOutCols / 2;
    const uint32_t stg = smem_u32(s_stage + ew * kStgBytes);
    const uint32_t my_srow = stg + lane * kStgPitch;
    TileCursor cur{segs, mp, NB};
    int i = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++i) {
      int4 seg;
      int m, nb;
      cur.seek(t, seg, m, nb);
      const int rows = min(kBM, seg.y - m * kBM);
      const int r_in_tile = q * 32 + lane;
      const bool valid = r_in_tile < rows;
      int64_t row = (int64_t)seg.x + m * kBM + r_in_tile;
      if (row_map != nullptr && valid) row = __ldg(row_map + row);
      const int64_t obase = row * ldo + (int64_t)nb * kOutCols + half * kHalfCols;  // element offset
      const int nvalid = max(0, min(32, rows - q * 32));                            // valid rows of this warp
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < kHalfCols; c0 += kStgCols) {
        uint32_t a[32], u[32];
        const int col = half * kHalfCols + c0;  // output column within the tile
        tmem_ld_32x32b_x32(taddr + col, a);
        if constexpr (kEpi == kEpiSwiGLU) tmem_ld_32x32b_x32(taddr + 128 + col, u);
        tmem_ld_wait();
        stage_row<kEpi>(my_srow, a, u);
        __syncwarp();
        // warp writes its 32 staged rows: 4 lanes x 16 B per row -> 8 rows per instruction
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rr = it * 8 + (lane >> 2);
          const int piece = lane & 3;
          const int64_t ob = __shfl_sync(0xffffffffu, obase, rr);
          if (rr < nvalid) {
            const uint4 v = ld_shared_v4(stg + rr * kStgPitch + piece * 16);
            st_global_v4(out + ob + c0 + piece * 8, v.x, v.y, v.z, v.w);
          }
        }
        __syncwarp();
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

// ==========================================================================================
// 2-CTA variant: a cluster of 2 CTAs (one TPC) computes 256 x 256 tiles with
// tcgen05.mma.cta_group::2 (UMMA M=256).  CTA r loads A rows [128r, 128r+128) and B rows
// (N) [128r, 128r+128) of the tile into its own smem; the leader (r=0) issues the MMAs,
// which read both CTAs' smem and write each CTA's 128 x 256 fp32 slice of D into its
// own TMEM.  Per CTA and k-block this moves 32 KB instead of 48 KB through L2 -> SMEM,
// and the freed smem buys 6 pipeline stages instead of 4.
//   full[s]   leader only: both CTAs' TMA count complete_tx bytes on it (peer via mapa)
//   empty[s]  per CTA: the leader's tcgen05.commit multicasts to both
//   tfull[a]  per CTA: multicast commit after the last k-block of a tile
//   tempty[a] leader only: 8 epilogue warps of each CTA arrive (peer remotely)
// Tiles are 256-row pair tiles of each segment; the cursor derives them from the
// 128-row prefix on the fly (pair tiles of a segment = ceil(m128 / 2)).  A segment whose
// 128-row tile count is odd ends in a half tile: M=128 cta_group::2 (64 rows per CTA, the
// "2x2" TMEM layout: row r in lanes r and 64 + r for the two column halves).
// Gather mode: 4 loader warps per CTA fill the A stage with 16-byte cp.async copies of
// x rows (manual 128B swizzle), the next tile's gather indices already in registers.
// ==========================================================================================
constexpr int k2Stages = 6;
constexpr uint32_t k2Half = 128 * kBK * 2;  // 16 KB: one CTA's half of A or of B per stage
constexpr size_t kGemm2Smem = 1024 + k2Stages * 2 * k2Half + 256 + kMaxSmemSegs * 20 + 16 + kEpiWarps * kStgBytes;

struct PairCursor {
  const int4* segs;
  const int* mp;  // 128-row tile prefix
  int NB;
  int s = 0;
  int base = 0;  // pair-tile index (x NB) where segment s starts
  __device__ __forceinline__ int pair_tiles(int i) const { return (mp[i + 1] - mp[i] + 1) >> 1; }
  // hf: the segment's last pair tile holds <= 128 rows (odd 128-row tile count) and runs as
  // an M=128 cta_group::2 MMA (64 rows per CTA) instead of a half-empty M=256 one
  __device__ __forceinline__ void seek(int t, int4& seg, int& m, int& nb, bool& hf) {
    int span = pair_tiles(s) * NB;
    while (base + span <= t) {
      base += span;
      ++s;
      span = pair_tiles(s) * NB;
    }
    seg = segs[s];
    const int ms = pair_tiles(s);
    const int local = t - base;
    // grouped rasterisation: groups of `gm` m-tiles; inside a group n-block-major, so the
    // pairs running side by side cover a gm x (pairs/gm) rectangle of the segment's tiles.
    // gm = 1: the NB pairs sharing an A tile run together and W stays L2-resident (small
    // experts); gm ~ sqrt(pairs): fewest DRAM bytes per wave when W does not fit L2.
    const int g = local / (gm * NB);
    const int gsz = min(gm, ms - g * gm);
    const int r = local - g * gm * NB;
    nb = r / gsz;
    m = g * gm + (r - nb * gsz);
    hf = half_tiles && m == ms - 1 && ((mp[s + 1] - mp[s]) & 1);
  }
  bool half_tiles = true;
  int gm = 1;
};

// kGather: the A tile is not TMA-loaded from a permuted buffer but gathered straight from
// the token activations by 4 extra "A-loader" warps with 16-byte cp.async (manual 128B
// swizzle), buffer row r reading token a_gather[r] / a_gather_div.  The copy of the
// scatter (K4) is never written.  Loader warps fence the generic-proxy writes for the
// tensor core (fence.proxy.async) and arrive on the leader's full barrier, which then
// counts 1 (B expect_tx) + 8 (4 loader warps x 2 CTAs) arrivals.
#ifndef HM_GEMM_ONCE_FIRST
#define HM_GEMM_ONCE_FIRST 1
#endif
#ifndef HM_ALOAD_WARPS
#define HM_ALOAD_WARPS 4
#endif
#ifndef HM_ALOOKAHEAD
#define HM_ALOOKAHEAD 2
#endif
constexpr int kALoadWarps = HM_ALOAD_WARPS;  // 4 or 8
constexpr int kALookahead = HM_ALOOKAHEAD;   // cp.async groups in flight per loader thread
constexpr int kARowsPerWarp = 128 / kALoadWarps;
constexpr int kARowsPerLane = kARowsPerWarp / 4;

__device__ __forceinline__ void cp_async16(uint32_t smem_dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// K6 fetch pairs (bounded expert cache; hm_fetch_plan in harmoe.h).  Thread 0 of each fetch CTA
// streams its share of a weight block (32 KB chunks, round-robin over the fetch CTAs) through a
// 6-stage shared-memory ring with TMA bulk copies: global -> smem completes on an mbarrier,
// smem -> global is a bulk-group store.  The last CTA to finish a block publishes the expert's
// ready flag (release) for the GEMM producers of the same launch.
// ------------------------------------------------------------------------------------------
constexpr int kFetchChunk = 32768;
constexpr int kFetchStages = 6;
static_assert(kFetchStages * kFetchChunk + 64 <= k2Stages * 2 * k2Half + 256, "fetch ring must fit the GEMM smem");

__device__ __forceinline__ void bulk_g2s(uint32_t smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_src), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// one weight block src -> dst (bytes % 16 == 0); this CTA copies chunks fc, fc + nf, ...
__device__ void fetch_block(uint8_t* dst, const uint8_t* src, long long bytes, uint32_t ring, uint64_t* bars,
                            uint32_t& par, int fc, int nf) {
  const long long nch = (bytes + kFetchChunk - 1) / kFetchChunk;
  const long long m = nch > fc ? (nch - fc + nf - 1) / nf : 0;
  auto issue = [&](long long i) {
    const int st = (int)(i % kFetchStages);
    const long long c = fc + i * nf;
    const uint32_t len = (uint32_t)min((long long)kFetchChunk, bytes - c * kFetchChunk);
    mbar_arrive_expect_tx(&bars[st], len);
    bulk_g2s(ring + st * kFetchChunk, src + c * kFetchChunk, len, &bars[st]);
  };
  // stage of chunk i is refilled (with chunk i + kFetchStages) kLag chunks later, once at most kLag
  // newer stores are still reading shared memory: loads and stores both stay in flight
  constexpr int kLag = 2;
  for (long long i = 0; i < min((long long)kFetchStages, m); ++i) issue(i);
  for (long long i = 0; i < m; ++i) {
    const int st = (int)(i % kFetchStages);
    mbar_wait(&bars[st], (par >> st) & 1u);
    par ^= 1u << st;
    const long long c = fc + i * nf;
    const uint32_t len = (uint32_t)min((long long)kFetchChunk, bytes - c * kFetchChunk);
    bulk_s2g(dst + c * kFetchChunk, ring + st * kFetchChunk, len);
    const long long j = i - kLag;  // chunk whose stage is refilled now
    if (j >= 0 && j + kFetchStages < m) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kLag) : "memory");
      issue(j + kFetchStages);
    }
  }
  for (long long j = max(0ll, m - kLag); j < m; ++j)  // refills the loop above did not reach
    if (j + kFetchStages < m) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      issue(j + kFetchStages);
    }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");  // bulk writes before the generic release
}

__device__ __forceinline__ void fetch_publish(int32_t* counter, int32_t* flag, int value, int nf) {
  __threadfence();
  if (atomicAdd(counter, 1) == nf - 1) {
    __threadfence();
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
  }
}

// the GEMM of this launch has finished every tile of expert e: 16 epilogue warps x pair tiles
__device__ void fetch_wait_done(const int32_t* done, const int4* segs, const int* mp, int n_seg, int e, int NB) {
  int pt = 0;
  for (int i = 0; i < n_seg; ++i)
    if (segs[i].w == e) pt += (mp[i + 1] - mp[i] + 1) >> 1;
  const int target = pt * NB * 16;
  long long spins = 0;
  while (ld_acquire_gpu(done + e) < target) {
    __nanosleep(256);
    if (++spins > (1ll << 25)) {  // watchdog (~10 s): never hang the device
      printf("hm grouped_gemm fetch pair: expert %d tiles never finished (%d < %d)\n", e, ld_acquire_gpu(done + e),
             target);
      __trap();
    }
  }
}

__device__ void fetch_pair_role(const hm_fetch_plan& fp, uint8_t* smem, int fc, int nf, const int4* segs,
                                const int* mp, int n_seg, int NB, const int32_t* done) {
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kFetchStages * kFetchChunk);
  if (threadIdx.x != 0) return;
  for (int st = 0; st < kFetchStages; ++st) mbar_init(&bars[st], 1);
  fence_mbar_init();
  const uint32_t ring = smem_u32(smem);
  uint32_t par = 0;
  const int n_fetch = *fp.n_fetch;
  const int C = fp.n_slots;
  if (2 * n_fetch > fp.n_counters) __trap();
  auto* dst_in = reinterpret_cast<uint8_t*>(fp.dst_in);
  auto* dst_out = reinterpret_cast<uint8_t*>(fp.dst_out);
  const long long inb = (long long)fp.in_bytes, outb = (long long)fp.out_bytes;
  if (fp.phase == 1) {
    for (int i = 0; i < n_fetch; ++i) {
      const int e = __ldg(fp.fetch + i);
      if (i >= C) fetch_wait_done(done, segs, mp, n_seg, __ldg(fp.fetch + i - C), NB);
      fetch_block(dst_in + (long long)(fp.first_slot + i % C) * inb,
                  reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(fp.src_in) + e)),
                  inb, ring, bars, par, fc, nf);
      fetch_publish(fp.counters + 2 * i, fp.ready_in + e, fp.value, nf);
    }
    for (int i = 0; i < min(C, n_fetch); ++i) {
      const int e = __ldg(fp.fetch + i);
      fetch_block(dst_out + (long long)(fp.first_slot + i) * outb,
                  reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(fp.src_out) + e)),
                  outb, ring, bars, par, fc, nf);
      fetch_publish(fp.counters + 2 * i + 1, fp.ready_out + e, fp.value, nf);
    }
  } else {
    for (int i = C; i < n_fetch; ++i) {
      const int e = __ldg(fp.fetch + i);
      fetch_wait_done(done, segs, mp, n_seg, __ldg(fp.fetch + i - C), NB);
      fetch_block(dst_out + (long long)(fp.first_slot + i % C) * outb,
                  reinterpret_cast<const uint8_t*>(__ldg(reinterpret_cast<const unsigned long long*>(fp.src_out) + e)),
                  outb, ring, bars, par, fc, nf);
      fetch_publish(fp.counters + 2 * i + 1, fp.ready_out + e, fp.value, nf);
    }
  }
}

// work unit t of the persistent walk -> pair tile + column slice (-1: the whole 256 columns)
struct TailSplit {
  int t_split;  // first split tile
  int units;    // walk length
  __device__ __forceinline__ int tile(int t, int& slice) const {
    if (t < t_split) {
      slice = -1;
      return t;
    }
    slice = (t - t_split) & 1;
    return t_split + ((t - t_split) >> 1);
  }
};

template <int kEpi, bool kGather>
__global__ void __launch_bounds__(kGather ? kGemmThreads + kALoadWarps * 32 : kGemmThreads, 1)
    grouped_gemm_2cta_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                             const __grid_constant__ CUtensorMap tmap_a64, const __grid_constant__ CUtensorMap tmap_b64,
                             int half_tiles /* bit0 half tiles, bits 1+: m-tile group of the walk */,
                             const int4* __restrict__ segs_g, const int* __restrict__ mprefix_g,
                             const int* __restrict__ n_seg_ptr, __nv_bfloat16* __restrict__ out, int N, int K,
                             int ldo, const int* __restrict__ row_map, const int* __restrict__ slot_ready,
                             int ready_from_slot, int epoch, const __nv_bfloat16* __restrict__ a_src,
                             const int* __restrict__ a_gather, int a_gather_div, int a_src_rows,
                             const unsigned long long* __restrict__ out_ptrs, const int* __restrict__ out_split,
                             int n_out, int* __restrict__ slot_done, const hm_fetch_plan fplan, int tail_split,
                             const CombineFuse cf, const int* __restrict__ a_arrive) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  if (fplan.pairs > 0 && (int)(blockIdx.x >> 1) >= (int)(gridDim.x >> 1) - fplan.pairs) {
    // K6 fetch pair: both CTAs of the cluster leave before any TMEM / cluster barrier
    const int fc = (int)blockIdx.x - ((int)gridDim.x - 2 * fplan.pairs);
    fetch_pair_role(fplan, smem, fc, 2 * fplan.pairs, reinterpret_cast<const int4*>(segs_g), mprefix_g, *n_seg_ptr,
                    N / kBN, slot_done);
    return;
  }
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + k2Stages * 2 * k2Half);
  uint64_t* empty = full + k2Stages;
  uint64_t* tfull = empty + k2Stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int4* s_segs = reinterpret_cast<int4*>(smem + k2Stages * 2 * k2Half + 256);
  int* s_mp = reinterpret_cast<int*>(s_segs + kMaxSmemSegs);
  uint8_t* s_stage = reinterpret_cast<uint8_t*>(s_mp + kMaxSmemSegs + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = (gridDim.x >> 1) - fplan.pairs;  // compute pairs (fetch pairs, if any, are the last)
  const int n_seg = *n_seg_ptr;
  const bool seg_in_smem = n_seg <= kMaxSmemSegs;
  if (seg_in_smem) {
    for (int i = threadIdx.x; i < n_seg; i += blockDim.x) s_segs[i] = segs_g[i];
    for (int i = threadIdx.x; i <= n_seg; i += blockDim.x) s_mp[i] = mprefix_g[i];
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full[s], kGather ? 1 + 2 * kALoadWarps : 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * kEpiWarps);
    }
    fence_mbar_init();
    if (!kGather) tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    if (half_tiles & 1) {
      if (!kGather) tma_prefetch_desc(&tmap_a64);
      if (kEpi == kEpiSwiGLU) tma_prefetch_desc(&tmap_b64);
    }
  }
  if (warp == 1) tmem_alloc_2cta<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // peer barriers initialised before any remote arrive / complete_tx
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int NB = N / kBN;
  const int4* segs = seg_in_smem ? s_segs : segs_g;
  const int* mp = seg_in_smem ? s_mp : mprefix_g;
  int total = 0;
  for (int i = lane; i < n_seg; i += 32) total += (mp[i + 1] - mp[i] + 1) >> 1;
  total = (int)__reduce_add_sync(0xffffffffu, (unsigned)total) * NB;
  const int KB = K / kBK;
  // Tail split: when the last wave is at most half full (rem = total % npairs <= npairs / 2,
  // e.g. Switch FFN2: 393 pair tiles on 74 pairs), its tiles run as two 128-column units on
  // twice as many pairs (N = 128 MMAs, 64 weight rows per CTA).  Every output element is still
  // one full-K accumulation in the same order: results are bit-identical to the unsplit walk.
  TailSplit ts{total, total};
  if (kEpi != kEpiSwiGLU && tail_split && slot_done == nullptr) {
    const int rem = total % npairs;
    if (rem > 0 && 2 * rem <= npairs) ts = TailSplit{total - rem, total + rem};
  }
  const int units = ts.units;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs) =====
      const uint64_t pol_a = l2_policy_evict_normal();
      const uint64_t pol_w = l2_policy_evict_last();
      // weights of a segment with a single pair m-tile are read once: streamed evict_first
      // (measured TMA read ceiling 6.0 vs 5.6 TB/s under evict_last, tools/stream_bench)
      const uint64_t pol_w1 = HM_GEMM_ONCE_FIRST ? l2_policy_evict_first() : pol_w;
      const uint32_t full_leader = mapa_shared(full, 0);
      PairCursor cur{segs, mp, NB};
      cur.half_tiles = (half_tiles & 1) != 0;
      cur.gm = max(1, half_tiles >> 1);
      int stage = 0;
      uint32_t phase = 0;
      int arrived_e = -1;
      for (int t = pair; t < units; t += npairs) {
        int4 seg;
        int m, nb, slice;
        bool hf;
        cur.seek(ts.tile(t, slice), seg, m, nb, hf);
        const int row0 = seg.x + m * 2 * kBM + (int)rank * (hf ? kBM / 2 : kBM);
        const int brow0 = seg.z * N + nb * kBN;
        // split unit: 128 columns, 64 weight rows per CTA (tmap_b64: 64-row boxes)
        const int brow = slice < 0 ? brow0 + (int)rank * (kBN / 2) : brow0 + slice * (kBN / 2) + (int)rank * (kBN / 4);
        // half tile: A is 64 rows per CTA; SwiGLU B is re-paired so CTA r holds gate rows
        // [64r, 64r+64) then the matching up rows -> every TMEM lane holds gate and up
        const bool b_split = hf && kEpi == kEpiSwiGLU;
        const uint32_t tx = (kGather ? 0u : (hf ? k2Half / 2 : k2Half)) + (slice < 0 ? k2Half : k2Half / 2);
        const uint64_t pol_b = cur.pair_tiles(cur.s) == 1 ? pol_w1 : pol_w;
        if (slot_ready != nullptr && seg.z >= ready_from_slot) {
          // watchdog: a fetch that never lands is a bug upstream; fail the launch instead of
          // hanging the device (~10 s)
#ifdef HM_DEBUG_K6
          printf("gemm pair %d rank %d tile %d: wait expert %d slot %d flag %d epoch %d\n", pair, rank, t, seg.w, seg.z,
                 ld_acquire_gpu(slot_ready + seg.w), epoch);
#endif
          long long spins = 0;
          while (ld_acquire_gpu(slot_ready + seg.w) < epoch) {
            __nanosleep(128);
            if (++spins > (1ll << 26)) {
              printf("hm grouped_gemm: fetched expert %d (slot %d) never became ready (%d < epoch %d)\n", seg.w,
                     seg.z, ld_acquire_gpu(slot_ready + seg.w), epoch);
              __trap();
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        if (a_arrive != nullptr && seg.w != arrived_e) {
          // expert-ordered dispatch (hm_dispatch_push_ordered): this segment's rows land over
          // NVLink while earlier segments compute; wait for all seg.y of them (system scope)
          long long spins = 0;
          while (ld_acquire_sys(a_arrive + seg.w) < seg.y) {
            __nanosleep(64);
            if (++spins > (1ll << 27)) {
              printf("hm grouped_gemm: rows of expert %d never arrived (%d < %d)\n", seg.w,
                     ld_acquire_sys(a_arrive + seg.w), seg.y);
              __trap();
            }
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          arrived_e = seg.w;
        }
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * tx);
          uint8_t* sa = smem + stage * 2 * k2Half;
          if (!kGather)
            tma_load_2d_2cta(sa, hf ? &tmap_a64 : &tmap_a, full_leader + stage * 8, kb * kBK, row0, pol_a);
          if (b_split) {
            tma_load_2d_2cta(sa + k2Half, &tmap_b64, full_leader + stage * 8, kb * kBK, brow0 + (int)rank * 64,
                             pol_b);
            tma_load_2d_2cta(sa + k2Half + k2Half / 2, &tmap_b64, full_leader + stage * 8, kb * kBK,
                             brow0 + kBN / 2 + (int)rank * 64, pol_b);
          } else {
            tma_load_2d_2cta(sa + k2Half, slice < 0 ? &tmap_b : &tmap_b64, full_leader + stage * 8, kb * kBK, brow,
                             pol_b);
          }
          if (++stage == k2Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (leader CTA) =====
      constexpr uint32_t idesc_full = make_idesc_bf16(2 * kBM, kBN);
      constexpr uint32_t idesc_half = make_idesc_bf16(kBM, kBN);  // 64 rows per CTA, "2x2" TMEM layout
      constexpr uint32_t idesc_full_n128 = make_idesc_bf16(2 * kBM, kBN / 2);  // tail-split units
      constexpr uint32_t idesc_half_n128 = make_idesc_bf16(kBM, kBN / 2);
      PairCursor cur{segs, mp, NB};
      cur.half_tiles = (half_tiles & 1) != 0;
      cur.gm = max(1, half_tiles >> 1);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = pair; t < units; t += npairs, ++i) {
        int4 seg;
        int m, nb, slice;
        bool hf;
        cur.seek(ts.tile(t, slice), seg, m, nb, hf);
        const uint32_t idesc =
            slice < 0 ? (hf ? idesc_half : idesc_full) : (hf ? idesc_half_n128 : idesc_full_n128);
        const int acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * 2 * k2Half);
          const uint64_t a0 = make_sdesc_sw128(sa);
          const uint64_t b0 = make_sdesc_sw128(sa + k2Half);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_2cta(d_tmem, a0 + (uint64_t)(k * 2), b0 + (uint64_t)(k * 2), idesc, (kb | k) != 0);
          umma_commit_2cta_multicast(&empty[stage], 0x3);
          if (++stage == k2Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2cta_multicast(&tfull[acc], 0x3);
      }
    }
  } else if (kGather && warp >= 2 + kEpiWarps) {
    // ===== A-loaders (gather mode): loader warp lw fills tile rows [32lw, 32lw+32); 8 lanes
    // copy one row's 128-byte k-block segment (16 B each), so every cp.async instruction
    // moves 4 whole rows = 4 full cache lines =====
    const int lw = warp - (2 + kEpiWarps);  // 0..kALoadWarps-1
    const int c = lane & 7;                 // 16-byte chunk of the row segment
    const int sub = lane >> 3;              // row within a group of 4
    const uint32_t full_leader = mapa_shared(full, 0);
    PairCursor cur{segs, mp, NB};
    cur.half_tiles = (half_tiles & 1) != 0;
    cur.gm = max(1, half_tiles >> 1);
    // the gather indices of a tile are loaded one tile ahead (software pipelined), so the
    // dependent index -> row address chain never stalls the first k-block of a tile
    auto tile_rows = [&](int tu, int& cta_rows, int (&gidx)[kARowsPerLane]) {
      int4 sg;
      int mm, nbb, sl;
      bool hff;
      cur.seek(ts.tile(tu, sl), sg, mm, nbb, hff);
      cta_rows = hff ? kBM / 2 : kBM;
      const int rows = max(0, min(cta_rows, sg.y - mm * 2 * kBM - (int)rank * cta_rows));
      const int rbase = sg.x + mm * 2 * kBM + (int)rank * cta_rows;
#pragma unroll
      for (int i = 0; i < kARowsPerLane; ++i) {
        const int r = lw * kARowsPerWarp + i * 4 + sub;
        gidx[i] = r < rows ? __ldg(a_gather + rbase + r) : 0;  // rows past the segment: any valid row
      }
    };
    int stage = 0, sig_stage = 0, pending = 0;
    uint32_t phase = 0;
    int cta_rows_nx = 0, gidx_nx[kARowsPerLane];
    if (pair < units) tile_rows(pair, cta_rows_nx, gidx_nx);
    for (int t = pair; t < units; t += npairs) {
      const int cta_rows = cta_rows_nx;
      const char* src[kARowsPerLane];
#pragma unroll
      for (int i = 0; i < kARowsPerLane; ++i) {
        const int src_row = min(gidx_nx[i] / a_gather_div, a_src_rows - 1);
        src[i] = reinterpret_cast<const char*>(a_src + (int64_t)src_row * K) + c * 16;
      }
      if (t + npairs < units) tile_rows(t + npairs, cta_rows_nx, gidx_nx);
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t dst = smem_u32(smem + stage * 2 * k2Half);
#pragma unroll
        for (int i = 0; i < kARowsPerLane; ++i) {
          const int r = lw * kARowsPerWarp + i * 4 + sub;
          if (r < cta_rows) cp_async16(dst + r * 128 + ((c ^ (r & 7)) << 4), src[i] + kb * 128);
        }
        cp_async_commit();
        if (++pending > kALookahead) {
          cp_async_wait<kALookahead>();
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(full_leader + sig_stage * 8);
          if (++sig_stage == k2Stages) sig_stage = 0;
          --pending;
        }
        if (++stage == k2Stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    __syncwarp();
    for (; pending > 0; --pending) {
      if (lane == 0) mbar_arrive_cluster(full_leader + sig_stage * 8);
      if (++sig_stage == k2Stages) sig_stage = 0;
    }
  } else {
    // ===== epilogue: warps 2..9 of both CTAs, each CTA drains its own 128 rows =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    constexpr int kOutCols = (kEpi == kEpiSwiGLU) ? kBN / 2 : kBN;
    constexpr int kHalfCols = kOutCols / 2;
    const uint32_t stg = smem_u32(s_stage + ew * kStgBytes);
    const uint32_t my_srow = stg + lane * kStgPitch;
    const uint32_t tempty_leader = mapa_shared(tempty, 0);
    PairCursor cur{segs, mp, NB};
    cur.half_tiles = (half_tiles & 1) != 0;
      cur.gm = max(1, half_tiles >> 1);
    int i = 0;
    for (int t = pair; t < units; t += npairs, ++i) {
      int4 seg;
      int m, nb, slice;
      bool hf;
      cur.seek(ts.tile(t, slice), seg, m, nb, hf);
      // Full tile: lane = row (128 per CTA), columns [0, 256).  Half tile (M=128 "2x2" layout):
      // row r < 64 of this CTA sits in lanes r (columns [0,128) of the MMA's N) and 64 + r
      // (columns [128,256)), both at TMEM columns [0,128).  SwiGLU half tiles were loaded
      // with B re-paired, so each lane half holds 64 gate columns then the 64 matching up.
      const int cta_rows = hf ? kBM / 2 : kBM;
      const int rows = max(0, min(cta_rows, seg.y - m * 2 * kBM - (int)rank * cta_rows));  // valid rows
      const int r_in_tile = (hf ? (q & 1) : q) * 32 + lane;
      // a split unit (never SwiGLU) is a 128-column tile: same layout at half the width
      const int hcols = slice < 0 ? kHalfCols : kHalfCols / 2;
      const int ncols = hf ? hcols / 2 : hcols;  // output columns of this warp
      const int tcol0 = half * ncols;            // its first TMEM column
      const int ocol0 = (slice < 0 ? 0 : slice * (kOutCols / 2)) + (hf ? (q >> 1) * hcols : 0) + half * ncols;
      const int upoff = hf ? kBN / 4 : kBN / 2;  // SwiGLU: TMEM column distance gate -> up
      const bool valid = r_in_tile < rows;
      int64_t row = (int64_t)seg.x + m * 2 * kBM + rank * cta_rows + r_in_tile;
      // remote output (EP over peer memory): rows go straight into their source rank's token-major
      // output over NVLink - per segment (source-major receive buffer: the source g whose range
      // [out_split[g], out_split[g+1]) holds the segment) or per row (expert-major receive buffer,
      // out_split == NULL: row_map carries (source << 24) | token-major row)
      __nv_bfloat16* obuf = out;
      if (out_ptrs != nullptr && out_split != nullptr) {
        int g = 0;
        while (g + 1 < n_out && __ldg(out_split + g + 1) <= seg.x) ++g;
        obuf = reinterpret_cast<__nv_bfloat16*>(__ldg(out_ptrs + g));
      }
      // the row-map load is issued here and first used after the accumulator wait below, so its
      // latency hides under the MMAs (ncu: its consumer was 4% of the epilogue's stall samples)
      if (row_map != nullptr && valid) row = __ldg(row_map + row);
      const bool direct = kEpi == kEpiStore && cf.y != nullptr && cf.k == 1;
      const int nvalid = max(0, min(32, rows - (r_in_tile - lane)));
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      if (row_map != nullptr && valid && out_ptrs != nullptr && out_split == nullptr) {
        obuf = reinterpret_cast<__nv_bfloat16*>(__ldg(out_ptrs + ((uint32_t)row >> 24)));
        row &= 0xFFFFFF;
      }
      // top-1 combine in the epilogue (cf.k == 1): row -> token t, y[t] = (residual[t] +) w[t] * Y,
      // the arithmetic of combine_dense_kernel (bit-identical), Y never written
      if (direct) obuf = reinterpret_cast<__nv_bfloat16*>(cf.y);
      // per-row output address (rows of one warp may belong to different ranks' buffers)
      const unsigned long long obase = reinterpret_cast<unsigned long long>(
          obuf + (row * ldo + (int64_t)nb * kOutCols + ocol0));
      float w_row = 0.0f;
      unsigned long long rbase = 0ull;
      if (direct && valid) {
        w_row = __ldg(cf.w + row);
        if (cf.residual != nullptr)
          rbase = reinterpret_cast<unsigned long long>(reinterpret_cast<const __nv_bfloat16*>(cf.residual) +
                                                       (row * ldo + (int64_t)nb * kOutCols + ocol0));
      }
      const uint32_t taddr = tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16);
      // the TMEM load of chunk c+1 is in flight while chunk c is stored, and the accumulator
      // is handed back to the MMA issuer as soon as its last columns are in registers (before
      // the last chunk's global stores)
      uint32_t a[32], u[32];
      tmem_ld_32x32b_x32(taddr + tcol0, a);
      if constexpr (kEpi == kEpiSwiGLU) tmem_ld_32x32b_x32(taddr + upoff + tcol0, u);
#pragma unroll 1
      for (int c0 = 0; c0 < ncols; c0 += kStgCols) {
        tmem_ld_wait();
        const bool last = c0 + kStgCols >= ncols;
        if (last) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
        }
        stage_row<kEpi>(my_srow, a, u);
        __syncwarp();
        if (!last) {
          const int col = tcol0 + c0 + kStgCols;
          tmem_ld_32x32b_x32(taddr + col, a);
          if constexpr (kEpi == kEpiSwiGLU) tmem_ld_32x32b_x32(taddr + upoff + col, u);
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rr = it * 8 + (lane >> 2);
          const int piece = lane & 3;
          const unsigned long long ob = __shfl_sync(0xffffffffu, obase, rr);
          if (direct) {
            const float wv = __shfl_sync(0xffffffffu, w_row, rr);
            const unsigned long long rb = __shfl_sync(0xffffffffu, rbase, rr);
            if (rr < nvalid) {
              const uint4 v = ld_shared_v4(stg + rr * kStgPitch + piece * 16);
              float acc[8];
              if (rb != 0ull) {
                const uint4 rv = ld_global_nc_v4(reinterpret_cast<const __nv_bfloat16*>(rb) + c0 + piece * 8);
                const uint32_t r4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  acc[2 * h] = bf16lo(r4[h]);
                  acc[2 * h + 1] = bf16hi(r4[h]);
                }
              } else {
#pragma unroll
                for (int h = 0; h < 8; ++h) acc[h] = 0.0f;
              }
              const uint32_t y4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                acc[2 * h] = __fadd_rn(acc[2 * h], __fmul_rn(wv, bf16lo(y4[h])));
                acc[2 * h + 1] = __fadd_rn(acc[2 * h + 1], __fmul_rn(wv, bf16hi(y4[h])));
              }
              st_global_v4(reinterpret_cast<__nv_bfloat16*>(ob) + c0 + piece * 8, pack_bf16x2(acc[0], acc[1]),
                           pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
            }
            continue;
          }
          if (rr < nvalid) {
            const uint4 v = ld_shared_v4(stg + rr * kStgPitch + piece * 16);
            st_global_v4(reinterpret_cast<__nv_bfloat16*>(ob) + c0 + piece * 8, v.x, v.y, v.z, v.w);
          }
        }
        __syncwarp();
      }
      if (kEpi == kEpiStore && cf.y != nullptr && !direct) {
        // fused combine: this warp's rows are stored for columns [nb*256 + ocol0, + ncols); each
        // (token, 64-column chunk) counts its k expert rows and the k-th arrival combines the
        // chunk in slot order - the arithmetic of combine_dense_kernel, so the output is
        // bit-identical to the separate combine.  Stores -> fence -> count (the last arriver
        // fences again before reading the other rows through L2).
        __threadfence();
        __syncwarp();
        const int kk = cf.k;
        const int nchk = ldo / 64;
        const int c64_0 = (nb * kOutCols + ocol0) / 64;
        const int tok = valid ? (int)(row / kk) : 0;
        for (int ch = 0; ch < ncols / 64; ++ch) {
          bool lastarr = false;
          if (valid)
            lastarr = atomicInc(cf.counters + (int64_t)tok * nchk + c64_0 + ch, (unsigned)(kk - 1)) ==
                      (unsigned)(kk - 1);
          uint32_t m = __ballot_sync(0xffffffffu, lastarr);
          if (m != 0u) __threadfence();
          while (m != 0u) {
            // up to 4 finished chunks per round, 8 lanes x 16 B per 64-column chunk
            uint32_t mm = m;
            int src = -1;
            for (int g = 0; g <= (lane >> 3); ++g) {
              src = (mm != 0u) ? __ffs(mm) - 1 : -1;
              mm &= mm - 1u;
            }
#pragma unroll
            for (int g = 0; g < 4; ++g) m &= m - 1u;
            const int t_c = __shfl_sync(0xffffffffu, tok, src < 0 ? 0 : src);
            if (src >= 0) {
              const int col = (c64_0 + ch) * 64 + (lane & 7) * 8;
              const __nv_bfloat16* yb = out + (int64_t)t_c * kk * ldo + col;
              float acc[8];
              if (cf.residual != nullptr) {
                const uint4 rv = ld_global_nc_v4(reinterpret_cast<const __nv_bfloat16*>(cf.residual) +
                                                 (int64_t)t_c * ldo + col);
                const uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  acc[2 * h] = bf16lo(rr[h]);
                  acc[2 * h + 1] = bf16hi(rr[h]);
                }
              } else {
#pragma unroll
                for (int h = 0; h < 8; ++h) acc[h] = 0.0f;
              }
              for (int j0 = 0; j0 < kk; j0 += 4) {
                uint4 u4[4];
                float wj[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  if (j0 + jj < kk) {
                    u4[jj] = ld_global_cg_v4(yb + (int64_t)(j0 + jj) * ldo);
                    wj[jj] = __ldg(cf.w + (int64_t)t_c * kk + j0 + jj);
                  }
                }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  if (j0 + jj < kk) {
                    const uint32_t uu[4] = {u4[jj].x, u4[jj].y, u4[jj].z, u4[jj].w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                      acc[2 * h] = __fadd_rn(acc[2 * h], __fmul_rn(wj[jj], bf16lo(uu[h])));
                      acc[2 * h + 1] = __fadd_rn(acc[2 * h + 1], __fmul_rn(wj[jj], bf16hi(uu[h])));
                    }
                  }
                }
              }
              st_global_v4(reinterpret_cast<__nv_bfloat16*>(cf.y) + (int64_t)t_c * ldo + col,
                           pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                           pack_bf16x2(acc[6], acc[7]));
            }
          }
        }
      }
      // K6 slot reuse: this warp is done with the tile, so its weight loads (TMA, consumed by
      // the MMAs before tfull fired) are complete; a fetch may overwrite a fetched expert's
      // cache slot once all 16 epilogue warps of all its tiles have counted here
      if (slot_done != nullptr && seg.z >= ready_from_slot && lane == 0) {
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(slot_done + seg.w) : "memory");
#ifdef HM_DEBUG_K6
        if (ew == 0 && rank == 0) printf("gemm pair %d tile %d: done expert %d\n", pair, t, seg.w);
#endif
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2cta<kTmemCols>(tmem_base);
  }
  // launched behind the ordered dispatch push (PDL): do not complete before it has, so the
  // stream order of later kernels covers the push too (returns at once without a dependency)
  if (a_arrive != nullptr) griddep_wait();
}

// ------------------------------------------------------------------------------------------
// Swap-AB 2-CTA grouped GEMM for weight-streaming shapes (tens of rows per expert: Switch-128,
// top-1).  The row-major kernel above puts the expert's token rows on the MMA's M (256 per pair,
// 128 at best with half tiles), so a 32-row expert drags 96+ padding rows of A through L2->SM
// per weight tile (355 of FFN1's 965 MB of L2->SM traffic at C1).  Here the MMA computes
// D^T = W . X^T: M = 256 weight rows (128 per CTA, TMA boxes of the B map above), N = 64 token
// rows (32 per CTA), so a 32-row expert pads to 64 token columns.  The epilogue transposes each
// warp's 32 features x 32 tokens through shared memory and writes token-major rows (ReLU, plain
// store, or the top-1 combine y[t] = (x[t] +) w[t] * Y with combine_dense_kernel's arithmetic).
// No gather, half tiles, fetch pairs or remote outputs (the LOCAL Switch path needs none).
// ------------------------------------------------------------------------------------------
#ifndef HM_SW_STAGES
#define HM_SW_STAGES 9
#endif
constexpr int kSwN = 64;                      // token rows per pair tile (MMA N)
constexpr uint32_t kSwBBytes = (kSwN / 2) * kBK * 2;  // 4 KB: one CTA's 32 token rows per stage
// a stage is 16 KB of weights + 4 KB of token rows (1 KB aligned for the 128-byte swizzle): 9
// stages fit where the row-major kernel keeps 6 of 32 KB, so more weight bytes are in flight
constexpr uint32_t kSwStage = k2Half + kSwBBytes;
constexpr int kSwStages = HM_SW_STAGES;
static_assert(kSwStages * kSwStage <= k2Stages * 2 * k2Half, "swap stages must fit the row-major layout");

template <int kEpi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_swap_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
                             const int4* __restrict__ segs_g, const int* __restrict__ n_seg_ptr,
                             __nv_bfloat16* __restrict__ out, int N, int K, int ldo, const int* __restrict__ row_map,
                             const CombineFuse cf) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSwStages * kSwStage);
  uint64_t* empty = full + kSwStages;
  uint64_t* tfull = empty + kSwStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int4* s_segs = reinterpret_cast<int4*>(smem + kSwStages * kSwStage + 256);
  int* s_tp = reinterpret_cast<int*>(s_segs + kMaxSmemSegs);  // [n_seg + 1] tile prefix
  uint8_t* s_stage = reinterpret_cast<uint8_t*>(s_tp + kMaxSmemSegs + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int n_seg = *n_seg_ptr;
  if (n_seg > kMaxSmemSegs) __trap();  // the segment table is staged in shared memory
  const int NB = N / kBN;
  for (int i = threadIdx.x; i < n_seg; i += blockDim.x) s_segs[i] = segs_g[i];
  __syncthreads();
  if (warp == 0) {  // tile prefix: token tiles of kSwN rows x NB weight blocks per segment
    int run = 0;
    for (int base = 0; base < n_seg; base += 32) {
      const int i = base + lane;
      const int x = i < n_seg ? ((s_segs[i].y + kSwN - 1) / kSwN) * NB : 0;
      int incl = x;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      if (i < n_seg) s_tp[i] = run + incl - x;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_tp[n_seg] = run;
  }
  if (warp == 0 && lane == 0) {
    for (int st = 0; st < kSwStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    for (int st = 0; st < 2; ++st) {
      mbar_init(&tfull[st], 1);
      mbar_init(&tempty[st], 2 * kEpiWarps);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
  }
  if (warp == 1) tmem_alloc_2cta<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = s_tp[n_seg];
  const int KB = K / kBK;
  // tile t -> (segment, token tile m, weight block nb); m-major inside a segment
  auto seek = [&](int t, int4& sg, int& m, int& nb) {
    int lo = 0, hi = n_seg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_tp[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    sg = s_segs[lo];
    const int loc = t - s_tp[lo];
    m = loc / NB;
    nb = loc - m * NB;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs): 128 weight rows + 32 token rows per stage =====
      const uint64_t pol_x = l2_policy_evict_last();
      const uint64_t pol_w_once = l2_policy_evict_first();
      const uint64_t pol_w = l2_policy_evict_last();
      const uint32_t full_leader = mapa_shared(full, 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < total; t += npairs) {
        int4 sg;
        int m, nb;
        seek(t, sg, m, nb);
        const int wrow = sg.z * N + nb * kBN + (int)rank * (kBN / 2);
        const int xrow = sg.x + m * kSwN + (int)rank * (kSwN / 2);
        const uint64_t pw = sg.y <= kSwN ? pol_w_once : pol_w;  // one token tile: weights read once
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (k2Half + kSwBBytes));
          uint8_t* sa = smem + stage * kSwStage;
          tma_load_2d_2cta(sa, &tmap_w, full_leader + stage * 8, kb * kBK, wrow, pw);
          tma_load_2d_2cta(sa + k2Half, &tmap_x, full_leader + stage * 8, kb * kBK, xrow, pol_x);
          if (++stage == kSwStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (leader CTA): M = 256 weight rows, N = 64 token rows =====
      constexpr uint32_t idesc = make_idesc_bf16(2 * kBM, kSwN);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int t = pair; t < total; t += npairs, ++i) {
        const int acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * kSwStage);
          const uint64_t a0 = make_sdesc_sw128(sa);
          const uint64_t b0 = make_sdesc_sw128(sa + k2Half);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16_2cta(d_tmem, a0 + (uint64_t)(k * 2), b0 + (uint64_t)(k * 2), idesc, (kb | k) != 0);
          umma_commit_2cta_multicast(&empty[stage], 0x3);
          if (++stage == kSwStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_2cta_multicast(&tfull[acc], 0x3);
      }
    }
  } else {
    // ===== epilogue: warp (q, half) drains features q*32.. of this CTA's 128, tokens half*32.. =====
    const int ew = warp - 2;
    const int q = warp & 3;
    const int half = ew >> 2;
    const uint32_t stg = smem_u32(s_stage + ew * kStgBytes);  // [32 tokens][kStgPitch]: 32 features
    const uint32_t tempty_leader = mapa_shared(tempty, 0);
    const bool direct = kEpi == kEpiStore && cf.y != nullptr && cf.k == 1;
    int i = 0;
    for (int t = pair; t < total; t += npairs, ++i) {
      int4 sg;
      int m, nb;
      seek(t, sg, m, nb);
      const int tok0 = m * kSwN + half * (kSwN / 2);  // first token of this warp within the segment
      // the 4 token rows this lane stores (it * 8 + lane / 4), their output rows loaded before the
      // accumulator wait
      int64_t orow[4];
      float wv[4];
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int tl = it * 8 + (lane >> 2);
        const bool ok = tok0 + tl < sg.y;
        int64_t r = (int64_t)sg.x + tok0 + tl;
        if (ok && row_map != nullptr) r = __ldg(row_map + r);
        orow[it] = ok ? r : -1;
        wv[it] = (direct && ok) ? __ldg(cf.w + r) : 0.0f;
      }
      const int acc = i & 1;
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      uint32_t a[32];
      tmem_ld_32x32b_x32(tmem_base + acc * kBN + ((uint32_t)(q * 32) << 16) + half * (kSwN / 2), a);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
      // transpose: feature `lane`, token j -> stg[j][lane]
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float v = __uint_as_float(a[j]);
        if constexpr (kEpi == kEpiRelu) v = fmaxf(v, 0.0f);
        const __nv_bfloat16 b = __float2bfloat16_rn(v);
        asm volatile("st.shared.b16 [%0], %1;" ::"r"(stg + j * kStgPitch + lane * 2),
                     "h"(*reinterpret_cast<const unsigned short*>(&b))
                     : "memory");
      }
      __syncwarp();
      const int col = nb * kBN + (int)rank * (kBN / 2) + q * 32 + (lane & 3) * 8;
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        if (orow[it] < 0) continue;
        const int tl = it * 8 + (lane >> 2);
        const uint4 v = ld_shared_v4(stg + tl * kStgPitch + (lane & 3) * 16);
        if (direct) {
          float accv[8];
          if (cf.residual != nullptr) {
            const uint4 rv = ld_global_nc_v4(reinterpret_cast<const __nv_bfloat16*>(cf.residual) + orow[it] * ldo + col);
            const uint32_t r4[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              accv[2 * h] = bf16lo(r4[h]);
              accv[2 * h + 1] = bf16hi(r4[h]);
            }
          } else {
#pragma unroll
            for (int h = 0; h < 8; ++h) accv[h] = 0.0f;
          }
          const uint32_t y4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            accv[2 * h] = __fadd_rn(accv[2 * h], __fmul_rn(wv[it], bf16lo(y4[h])));
            accv[2 * h + 1] = __fadd_rn(accv[2 * h + 1], __fmul_rn(wv[it], bf16hi(y4[h])));
          }
          st_global_v4(reinterpret_cast<__nv_bfloat16*>(cf.y) + orow[it] * ldo + col, pack_bf16x2(accv[0], accv[1]),
                       pack_bf16x2(accv[2], accv[3]), pack_bf16x2(accv[4], accv[5]), pack_bf16x2(accv[6], accv[7]));
        } else {
          st_global_v4(out + orow[it] * ldo + col, v.x, v.y, v.z, v.w);
        }
      }
      __syncwarp();
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2cta<kTmemCols>(tmem_base);
  }
}

static bool use_half_tiles() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HM_GEMM_NO_HALF");
    v = (e != nullptr && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// tail split of a half-empty last wave into 128-column units (HM_GEMM_TAIL_SPLIT=0 disables)
static bool use_tail_split() {
  const char* e = getenv("HM_GEMM_TAIL_SPLIT");  // read per launch: tests compare both walks
  return !(e != nullptr && e[0] == '0');
}

// m-tile group of the pair-tile walk: 1 when a segment's weights (N x K bf16) fit easily
// in L2 (they stay resident while the A tiles stream once: Qwen-128 / Switch-128, +2% FFN1
// over the n-block-major walk), else 16 m-tiles per group (Mixtral 8x7B, 235 MB of W1 per
// expert: 1.54 -> 1.72-1.80 Mtok/s vs gm = 1, best of the 1/4/8/16/24/32/64 sweep within
// the power-cap noise).  HM_GEMM_GM overrides.
static int walk_group(int N, int K) {
  const char* e = getenv("HM_GEMM_GM");
  if (e != nullptr && atoi(e) > 0) return atoi(e);
  return ((size_t)N * K * 2 <= (size_t)24 << 20) ? 1 : 16;
}

static bool use_2cta() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HM_GEMM_1CTA");
    v = (e != nullptr && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

// Co-resident CTA pairs of the 2-CTA kernel (cudaOccupancyMaxActiveClusters for its cluster
// shape, block and smem), cached per device and variant.  The persistent walk assigns tiles to
// pairs statically, so launching more pairs than can be resident would leave the extra pairs'
// tiles waiting for a whole pair to retire - and deadlock a GEMM that waits on a concurrent
// kernel (bounded-cache K6).
template <int kEpi, bool kGather>
static int resident_pairs_of() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    cudaFuncSetAttribute(grouped_gemm_2cta_kernel<kEpi, kGather>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGemm2Smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(num_sms() & ~1));
    cfg.blockDim = dim3(kGemmThreads + (kGather ? kALoadWarps * 32 : 0));
    cfg.dynamicSmemBytes = kGemm2Smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, grouped_gemm_2cta_kernel<kEpi, kGather>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    cache[dev] = n;
  }
  return cache[dev];
}

int launch_grouped_gemm_swap(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                             const int32_t* segs, const int32_t* n_seg, int epilogue, void* out, const int32_t* row_map,
                             const CombineFuse* combine, cudaStream_t stream) {
  if (N % kBN != 0 || K % kBK != 0 || N <= 0 || K <= 0)
    return set_error(HM_EINVAL, "grouped_gemm_swap: N %% 256 and K %% 64 must be 0");
  if (w_rows % N != 0) return set_error(HM_EINVAL, "grouped_gemm_swap: weight rows must be a multiple of N");
  if (epilogue != kEpiStore && epilogue != kEpiRelu)
    return set_error(HM_EINVAL, "grouped_gemm_swap: STORE or RELU epilogue only");
  CombineFuse cf = {};
  if (combine != nullptr && combine->y != nullptr) {
    cf = *combine;
    if (epilogue != kEpiStore || cf.k != 1 || cf.w == nullptr || row_map == nullptr)
      return set_error(HM_EINVAL, "grouped_gemm_swap: the fused combine is the top-1 one (STORE, k = 1, row map)");
  } else if (out == nullptr) {
    return set_error(HM_EINVAL, "grouped_gemm_swap: out is required");
  }
  if (a_rows <= 0) return HM_OK;
  CUtensorMap tw, tx;
  int rc = make_tmap_2d_bf16(&tw, W, (uint64_t)w_rows, (uint64_t)K, kBN / 2, kBK);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tx, A, (uint64_t)a_rows, (uint64_t)K, kSwN / 2, kBK);
  if (rc) return rc;
  const int pairs = min(num_sms() / 2, gemm_resident_pairs(epilogue, false));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = kGemm2Smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int4* s4 = reinterpret_cast<const int4*>(segs);
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  cudaError_t e;
  if (epilogue == kEpiRelu) {
    cudaFuncSetAttribute(grouped_gemm_swap_kernel<kEpiRelu>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGemm2Smem);
    e = cudaLaunchKernelEx(&cfg, grouped_gemm_swap_kernel<kEpiRelu>, tw, tx, s4, n_seg, o, N, K, N, row_map, cf);
  } else {
    cudaFuncSetAttribute(grouped_gemm_swap_kernel<kEpiStore>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGemm2Smem);
    e = cudaLaunchKernelEx(&cfg, grouped_gemm_swap_kernel<kEpiStore>, tw, tx, s4, n_seg, o, N, K, N, row_map, cf);
  }
  if (e != cudaSuccess) return set_error(HM_ECUDA, "grouped_gemm_swap launch: %s", cudaGetErrorString(e));
  return check_launch("grouped_gemm_swap");
}

int gemm_resident_pairs(int epilogue, bool gather) {
  switch (epilogue * 2 + (gather ? 1 : 0)) {
    case kEpiStore * 2: return resident_pairs_of<kEpiStore, false>();
    case kEpiStore * 2 + 1: return resident_pairs_of<kEpiStore, true>();
    case kEpiRelu * 2: return resident_pairs_of<kEpiRelu, false>();
    case kEpiRelu * 2 + 1: return resident_pairs_of<kEpiRelu, true>();
    case kEpiSwiGLU * 2: return resident_pairs_of<kEpiSwiGLU, false>();
    case kEpiSwiGLU * 2 + 1: return resident_pairs_of<kEpiSwiGLU, true>();
    default: return -1;
  }
}

int launch_grouped_gemm(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                        const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue,
                        void* out, const int32_t* row_map, const int32_t* a_gather, int a_gather_div,
                        const int32_t* slot_ready, int ready_from_slot, int epoch, cudaStream_t stream,
                        const unsigned long long* out_ptrs, const int32_t* out_split, int n_out, int32_t* slot_done,
                        const hm_fetch_plan* fetch, const CombineFuse* combine, const int32_t* a_arrive, int pdl) {
  if (N % kBN != 0 || K % kBK != 0 || N <= 0 || K <= 0)
    return set_error(HM_EINVAL, "grouped_gemm: N %% 256 and K %% 64 must be 0");
  if (w_rows % N != 0) return set_error(HM_EINVAL, "grouped_gemm: weight rows must be a multiple of N");
  if (a_gather != nullptr && a_gather_div < 1) return set_error(HM_EINVAL, "grouped_gemm: a_gather_div must be >= 1");
  if (out_ptrs != nullptr && (n_out < 1 || n_out > 256 || (out_split == nullptr && row_map == nullptr)))
    return set_error(HM_EINVAL, "grouped_gemm: remote output needs n_out in [1, 256] and out_split or a tagged row_map");
  if (out_ptrs != nullptr && !use_2cta())
    return set_error(HM_EINVAL, "grouped_gemm: remote output needs the 2-CTA kernel (unset HM_GEMM_1CTA)");
  if (slot_done != nullptr && !use_2cta())
    return set_error(HM_EINVAL, "grouped_gemm: slot_done counters need the 2-CTA kernel (unset HM_GEMM_1CTA)");
  hm_fetch_plan fplan = {};
  if (fetch != nullptr) {
    fplan = *fetch;
    if (slot_done == nullptr || !use_2cta())
      return set_error(HM_EINVAL, "grouped_gemm: fetch pairs need slot_done and the 2-CTA kernel");
    if (fplan.pairs < 1 || (fplan.phase != 1 && fplan.phase != 2) || fplan.n_slots < 1 || fplan.fetch == nullptr ||
        fplan.n_fetch == nullptr || fplan.src_in == nullptr || fplan.src_out == nullptr || fplan.ready_in == nullptr ||
        fplan.ready_out == nullptr || fplan.counters == nullptr || fplan.n_counters < 2 ||
        fplan.in_bytes % 16 != 0 || fplan.out_bytes % 16 != 0)
      return set_error(HM_EINVAL, "grouped_gemm: incomplete fetch plan");
    const cudaError_t me = cudaMemsetAsync(fplan.counters, 0, sizeof(int32_t) * fplan.n_counters, stream);
    if (me != cudaSuccess) return set_error(HM_ECUDA, "grouped_gemm fetch counters: %s", cudaGetErrorString(me));
  }
  CombineFuse cf = {};
  if (combine != nullptr && combine->y != nullptr) {
    cf = *combine;
    if (epilogue != kEpiStore || row_map == nullptr || out_ptrs != nullptr || (out == nullptr && cf.k != 1) ||
        !use_2cta() || cf.w == nullptr || (cf.counters == nullptr && cf.k != 1) || cf.k < 1 || cf.k > 32 || N % 64 != 0)
      return set_error(HM_EINVAL, "grouped_gemm: the fused combine needs the STORE epilogue with a token-major "
                                  "row map, local output, weights, counters and 1 <= k <= 32");
  }
  if (a_arrive != nullptr && (a_gather != nullptr || !use_2cta()))
    return set_error(HM_EINVAL, "grouped_gemm: arrival waits need TMA-loaded A rows and the 2-CTA kernel");
  if (a_rows <= 0) return HM_OK;
  CUtensorMap ta, tb;
  // gathered A: 1-row boxes fetched four at a time by tile::gather4
  int rc = make_tmap_2d_bf16(&ta, A, (uint64_t)a_rows, (uint64_t)K, a_gather != nullptr ? 1 : kBM, kBK);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tb, W, (uint64_t)w_rows, (uint64_t)K, kBN, kBK);
  if (rc) return rc;
  const int ldo = (epilogue == kEpiSwiGLU) ? N / 2 : N;
  const int grid = num_sms();
  const int4* s4 = reinterpret_cast<const int4*>(segs);
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  if (use_2cta()) {
    CUtensorMap tb2;  // each CTA of the pair loads 128 of the tile's 256 weight rows
    rc = make_tmap_2d_bf16(&tb2, W, (uint64_t)w_rows, (uint64_t)K, kBN / 2, kBK);
    if (rc) return rc;
    // half tiles: 64-row A boxes, and 64-row B boxes for the re-paired SwiGLU weight halves
    const int half_tiles = (use_half_tiles() ? 1 : 0) | (walk_group(N, K) << 1);  // tile-walk flags
    CUtensorMap ta64 = ta, tb64 = tb2;
    if ((half_tiles & 1) && a_gather == nullptr) {
      rc = make_tmap_2d_bf16(&ta64, A, (uint64_t)a_rows, (uint64_t)K, kBM / 2, kBK);
      if (rc) return rc;
    }
    // 64-row weight boxes: SwiGLU half tiles, and the 128-column units of the tail split
    rc = make_tmap_2d_bf16(&tb64, W, (uint64_t)w_rows, (uint64_t)K, kBN / 4, kBK);
    if (rc) return rc;
    // (not with the fused combine: its 64-column chunk counters assume >= 64-column warp spans)
    const int tail_split =
        (epilogue != kEpiSwiGLU && slot_done == nullptr && cf.y == nullptr && use_tail_split()) ? 1 : 0;
    const bool gather = a_gather != nullptr;
    // every pair resident at once (static tile walk; the fetch pairs and the compute pairs wait
    // on each other); fetch pairs come out of the same budget
    const int pairs = min(num_sms() / 2, gemm_resident_pairs(epilogue, gather));
    if (pairs - fplan.pairs < 1) return set_error(HM_EINVAL, "grouped_gemm: no compute pair left beside the fetch pairs");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    cfg.blockDim = dim3(kGemmThreads + (gather ? kALoadWarps * 32 : 0));
    cfg.dynamicSmemBytes = kGemm2Smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: start behind the push
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    cudaError_t e = cudaSuccess;
    const auto* a_src = reinterpret_cast<const __nv_bfloat16*>(A);
#define HM_GEMM2(EPI, G)                                                                                          \
  do {                                                                                                            \
    cudaFuncSetAttribute(grouped_gemm_2cta_kernel<EPI, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                         (int)kGemm2Smem);                                                                        \
    e = cudaLaunchKernelEx(&cfg, grouped_gemm_2cta_kernel<EPI, G>, ta, tb2, ta64, tb64, half_tiles, s4,          \
                           mtile_prefix, n_seg, o, N, K,                                                          \
                           ldo, row_map, slot_ready, ready_from_slot, epoch, a_src, a_gather, a_gather_div,       \
                           (int)a_rows, out_ptrs, out_split, n_out, slot_done, fplan, tail_split, cf, a_arrive);  \
  } while (0)
    switch (epilogue * 2 + (gather ? 1 : 0)) {
      case kEpiStore * 2: HM_GEMM2(kEpiStore, false); break;
      case kEpiStore * 2 + 1: HM_GEMM2(kEpiStore, true); break;
      case kEpiRelu * 2: HM_GEMM2(kEpiRelu, false); break;
      case kEpiRelu * 2 + 1: HM_GEMM2(kEpiRelu, true); break;
      case kEpiSwiGLU * 2: HM_GEMM2(kEpiSwiGLU, false); break;
      case kEpiSwiGLU * 2 + 1: HM_GEMM2(kEpiSwiGLU, true); break;
      default: return set_error(HM_EINVAL, "grouped_gemm: unknown epilogue");
    }
#undef HM_GEMM2
    if (e != cudaSuccess) return set_error(HM_ECUDA, "grouped_gemm (2-CTA) launch: %s", cudaGetErrorString(e));
    return check_launch("grouped_gemm_2cta");
  }
  if (cf.y != nullptr) return set_error(HM_EINVAL, "grouped_gemm: the fused combine needs the 2-CTA kernel");
#define HM_GEMM(EPI)                                                                                         \
  do {                                                                                                       \
    cudaFuncSetAttribute(grouped_gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem); \
    grouped_gemm_kernel<EPI><<<grid, kGemmThreads, kGemmSmem, stream>>>(                                    \
        ta, tb, s4, mtile_prefix, n_seg, o, N, K, ldo, row_map, a_gather, a_gather_div, (int)a_rows,        \
        slot_ready, ready_from_slot, epoch);                                                                \
  } while (0)
  switch (epilogue) {
    case kEpiStore: HM_GEMM(kEpiStore); break;
    case kEpiRelu: HM_GEMM(kEpiRelu); break;
    case kEpiSwiGLU: HM_GEMM(kEpiSwiGLU); break;
    default: return set_error(HM_EINVAL, "grouped_gemm: unknown epilogue");
  }
#undef HM_GEMM
  return check_launch("grouped_gemm");
}

}  // namespace hm
