// K3: HarMoEny scheduler on the GPU, plus the dispatch/GEMM layout it implies.
//
// dev_schedule restates moesim/policies.py:109-141 (initial_assign +
// _rebalance_core, Alg. 2 of PAPER.md:702-745) bit for bit:
//   t_avg = floor(sum S / G); while any t_g > t_avg:
//     g_max = argmax t; g_from = argmax_g sum_e S[g,e,g_max];
//     e_max = argmax_e S[g_from,e,g_max]; stop if that bucket < q;
//     g_min = argmin t; stop if g_min == g_max or t[g_min] + q > t_avg;
//     move min(bucket, t_avg - t[g_min]) tokens (g_from,e_max): g_max -> g_min.
// All argmax/argmin ties break to the lowest index (numpy first occurrence).
// One CTA; S lives in shared memory (32 KB at G=8, E=128); the serial loop runs
// in a single warp with warp-shuffle argmax (lane d owns t[d]; flows F[g][d] are
// kept incrementally so g_from is one lane-parallel read).
//
// dev_layout turns S into (a) slot_base[g,e,d], the buffer row of the first
// token of every bucket, and (b) the grouped GEMM's segment list in the
// per-GPU execution order of plan_gpu_execution (engine.py:233-234: resident
// experts with work by (-tokens, e), then fetched experts by (-tokens, e)).
//
// plan_kernel fuses the whole planning stage into one launch: per-rank
// histogram + per-tile offsets from the router's tile histograms (LOCAL) or the
// all-gathered m_all (EP), the schedule, and the layout.
#include <climits>

#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

constexpr int kPlanThreads = 1024;
constexpr int kLayMaxGE = 8192;  // G*E entries kept in smem by the layout

// phase timestamps of the last plan_kernel (diagnostics: hm_debug_plan_phases)
__device__ unsigned long long g_phase_ns[8];

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// %globaltimer phase stamps (hm_debug_plan_phases) only in a diagnostics build (-DHM_PLAN_PHASES,
// tools/plan_phases*.py): the reads cost the production planner ~1.6 us per launch (Switch C1
// router + planner + scatter stage 30.3 -> 28.7 us without them)
#ifdef HM_PLAN_PHASES
#define HM_PHASE(i) g_phase_ns[i] = globaltimer_ns()
#else
#define HM_PHASE(i) \
  do {              \
  } while (0)
#endif

int read_plan_phases(long long* out8) {
  unsigned long long h[8];
  const cudaError_t e = cudaMemcpyFromSymbol(h, g_phase_ns, sizeof(h));
  if (e != cudaSuccess) return set_error(HM_ECUDA, "read plan phases: %s", cudaGetErrorString(e));
  for (int i = 0; i < 8; ++i) out8[i] = (long long)h[i];
  return HM_OK;
}

// diagnostics build only (-DHM_PLAN_STAMPS, tools/plan_clocks.py): clock64 at block-wide barriers
#ifdef HM_PLAN_STAMPS
__device__ long long g_pclk[16];
#define HM_PSTAMP(i)                                   \
  do {                                                 \
    __syncthreads();                                   \
    if (threadIdx.x == 0) g_pclk[i] = clock64();       \
  } while (0)
extern "C" __attribute__((visibility("default"))) int hm_debug_plan_clocks(long long* out16) {
  return cudaMemcpyFromSymbol(out16, g_pclk, sizeof(long long) * 16) == cudaSuccess ? 0 : 1;
}
#else
#define HM_PSTAMP(i) \
  do {               \
  } while (0)
#endif

__device__ __forceinline__ void warp_argmax_ll(long long& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const long long ov = __shfl_xor_sync(0xffffffffu, v, off);
    const int oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

__device__ __forceinline__ void warp_argmin_ll(long long& v, int& i) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const long long ov = __shfl_xor_sync(0xffffffffu, v, off);
    const int oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (ov < v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

// ------------------------------------------------------------------------------------------
// histogram reduce: m_all[r][e] = sum_tiles tile_hist, tile_off = exclusive prefix over tiles
// (all threads of the block; 8 tile-chunks per expert lane, coalesced over experts)
// ------------------------------------------------------------------------------------------
__device__ void dev_hist_reduce(const int32_t* __restrict__ tile_hist, int n_ranks, int tpr, int E,
                                int* m_out /* smem or global [n_ranks*E] */, int32_t* __restrict__ m_global,
                                int32_t* __restrict__ tile_off, int* s_part /* [8*128] */) {
  const int tid = threadIdx.x;
  const int el = tid & 127, sub = tid >> 7;  // 8 sub-chunks x 128 experts (blockDim = 1024)
  if (n_ranks >= 2 && tpr <= 32) {
    // few tiles per rank: the 8 thread groups take whole ranks, each thread scans one expert
    for (int r = sub; r < n_ranks; r += 8)
      for (int e = el; e < E; e += 128) {
        int run = 0;
#pragma unroll 4
        for (int m = 0; m < tpr; ++m) {
          const int64_t i = ((int64_t)r * tpr + m) * E + e;
          const int v = tile_hist[i];
          tile_off[i] = run;
          run += v;
        }
        m_out[r * E + e] = run;
        if (m_global != nullptr) m_global[r * E + e] = run;
      }
    __syncthreads();
    return;
  }
  const int chunk = (tpr + 7) / 8;
  if (chunk <= 16) {
    // one batch of independent loads per thread (one memory round trip instead of a chain)
    for (int r = 0; r < n_ranks; ++r)
      for (int e0 = 0; e0 < E; e0 += 128) {
        const int e = e0 + el;
        const int m_lo = min(tpr, sub * chunk), m_hi = min(tpr, m_lo + chunk);
        int v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          v[j] = (e < E && m_lo + j < m_hi) ? tile_hist[((int64_t)r * tpr + m_lo + j) * E + e] : 0;
        int sum = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) sum += v[j];
        s_part[sub * 128 + el] = sum;
        __syncthreads();
        if (e < E) {
          int run = 0;
          for (int s = 0; s < sub; ++s) run += s_part[s * 128 + el];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (m_lo + j < m_hi) {
              tile_off[((int64_t)r * tpr + m_lo + j) * E + e] = run;
              run += v[j];
            }
          if (sub == 7) {
            int total = 0;
            for (int s = 0; s < 8; ++s) total += s_part[s * 128 + el];
            m_out[r * E + e] = total;
            if (m_global != nullptr) m_global[r * E + e] = total;
          }
        }
        __syncthreads();
      }
    return;
  }
  for (int r = 0; r < n_ranks; ++r) {
    for (int e0 = 0; e0 < E; e0 += 128) {
      const int e = e0 + el;
      const int m_lo = min(tpr, sub * chunk), m_hi = min(tpr, m_lo + chunk);
      int sum = 0;
      if (e < E) {
#pragma unroll 4
        for (int m = m_lo; m < m_hi; ++m) sum += tile_hist[((int64_t)r * tpr + m) * E + e];
      }
      s_part[sub * 128 + el] = sum;
      __syncthreads();
      if (e < E) {
        int base = 0;
        for (int s = 0; s < sub; ++s) base += s_part[s * 128 + el];
        int run = base;
#pragma unroll 4
        for (int m = m_lo; m < m_hi; ++m) {
          const int64_t i = ((int64_t)r * tpr + m) * E + e;
          const int v = tile_hist[i];
          tile_off[i] = run;
          run += v;
        }
        if (sub == 7) {
          m_out[r * E + e] = run;
          if (m_global != nullptr) m_global[r * E + e] = run;
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------------------------
// schedule (initial_assign + rebalance); S may live in smem or global memory
// ------------------------------------------------------------------------------------------
// Fast rebalance loop: every count < 2^21, so (value, index) pairs pack into 32-bit keys
// and each argmax/argmin is ONE warp redux (lowest index wins ties: the index is stored
// inverted for max, plain for min).  St is S transposed to [g][d][e] so the e_max scan
// reads consecutive words.  Same decisions as the 64-bit loop below (and the reference).
__device__ int rebalance_fast(int* S, int* St, long long* F, int G, int E, int q, int lane, int& t_lane,
                              int t_avg) {
  int t = t_lane;
  int iters = 0;
  for (;;) {
    if (__ballot_sync(0xffffffffu, lane < G && t > t_avg) == 0u) break;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, lane < G ? ((unsigned)t << 5) | (31u - lane) : 0u);
    const int g_max = 31 - (int)(kmax & 31u);
    const unsigned kf =
        __reduce_max_sync(0xffffffffu, lane < G ? ((unsigned)F[lane * 32 + g_max] << 5) | (31u - lane) : 0u);
    const int g_from = 31 - (int)(kf & 31u);
    const int* col = St + (g_from * G + g_max) * E;
    unsigned kb = 0u;
    for (int e = lane; e < E; e += 32) kb = max(kb, ((unsigned)col[e] << 10) | (1023u - e));
    kb = __reduce_max_sync(0xffffffffu, kb);
    const int t_move = (int)(kb >> 10);
    const int e_max = 1023 - (int)(kb & 1023u);
    if (t_move < q) break;
    const unsigned kmin = __reduce_min_sync(0xffffffffu, lane < G ? ((unsigned)t << 5) | lane : 0xffffffffu);
    const int g_min = (int)(kmin & 31u);
    const int vmin = (int)(kmin >> 5);
    if (g_min == g_max || (long long)vmin + q > t_avg) break;
    const int t_s = min(t_move, t_avg - vmin);
    if (lane == 0) {
      S[(g_from * E + e_max) * G + g_max] -= t_s;
      S[(g_from * E + e_max) * G + g_min] += t_s;
      St[(g_from * G + g_max) * E + e_max] -= t_s;
      St[(g_from * G + g_min) * E + e_max] += t_s;
      F[g_from * 32 + g_max] -= t_s;
      F[g_from * 32 + g_min] += t_s;
    }
    if (lane == g_max) t -= t_s;
    if (lane == g_min) t += t_s;
    __syncwarp();
    ++iters;
  }
  t_lane = t;
  return iters;
}

__device__ void dev_schedule(int* S, bool init_from_m, const int* m_all, const int* home, int G, int E, int q,
                             int rebalance, int32_t* iters_out, int32_t* loads_out, long long* F /* [32*32] */,
                             int* St = nullptr /* [G*G*E] scratch for the fast loop */) {
  const int n = G * E * G;
  if (init_from_m) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) S[i] = 0;
    __syncthreads();
    if (rebalance == HM_POLICY_EVEN_SPLIT) {
      // even_split_assign (policies.py:174-203): expert e's pooled total split as evenly as
      // integers allow (remainder to the lowest-index GPUs), sources fill the per-GPU targets
      // in index order.  One thread per expert; at most 2G-1 (source, dest) steps.
      for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int total = 0;
        for (int g = 0; g < G; ++g) total += m_all[g * E + e];
        if (total == 0) continue;
        const int base = total / G, rem = total - base * G;
        int dest = 0;
        int room = base + (0 < rem ? 1 : 0);
        for (int src = 0; src < G; ++src) {
          int left = m_all[src * E + e];
          while (left > 0) {
            while (room == 0) {
              ++dest;
              room = base + (dest < rem ? 1 : 0);
            }
            const int take = min(left, room);
            S[(src * E + e) * G + dest] += take;
            room -= take;
            left -= take;
          }
        }
      }
    } else {
      for (int i = threadIdx.x; i < G * E; i += blockDim.x) {
        const int g = i / E, e = i - (i / E) * E;
        S[(g * E + e) * G + home[e]] = m_all[i];
      }
    }
    if (rebalance != HM_POLICY_REBALANCE) rebalance = HM_POLICY_NONE;
  }
  __syncthreads();
  // flows F[g][d] = sum_e S[g,e,d]: one warp per (g, d) pair, lanes stride the experts
  {
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int i = threadIdx.x >> 5; i < G * G; i += nw) {
      const int g = i / G, d = i - (i / G) * G;
      long long f = 0;
      for (int e = lane; e < E; e += 32) f += S[(g * E + e) * G + d];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) f += __shfl_xor_sync(0xffffffffu, f, off);
      if (lane == 0) F[g * 32 + d] = f;
    }
  }
  if (St != nullptr && rebalance) {  // St[g][d][e]: one warp per (g, d) row, lanes stride the experts
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int row = threadIdx.x >> 5; row < G * G; row += nw) {
      const int g = row / G, d = row - g * G;
      for (int e = lane; e < E; e += 32) St[row * E + e] = S[(g * E + e) * G + d];
    }
  }
  __syncthreads();
  HM_PSTAMP(2);

  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long t = 0;
    if (lane < G)
      for (int g = 0; g < G; ++g) t += F[g * 32 + lane];
    long long total = (lane < G) ? t : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(0xffffffffu, total, off);
    const long long t_avg = total / G;
    int iters = 0;
    if (rebalance && St != nullptr && total < (1ll << 21) && E <= 1024) {
      int ti = (int)t;
      iters = rebalance_fast(S, St, F, G, E, q, lane, ti, (int)t_avg);
      t = ti;
    } else if (rebalance) {
      for (;;) {
        const unsigned over = __ballot_sync(0xffffffffu, lane < G && t > t_avg);
        if (over == 0u) break;
        long long vmax = (lane < G) ? t : LLONG_MIN;
        int g_max = lane;
        warp_argmax_ll(vmax, g_max);
        long long fv = (lane < G) ? F[lane * 32 + g_max] : LLONG_MIN;
        int g_from = lane;
        warp_argmax_ll(fv, g_from);
        long long best = LLONG_MIN;
        int e_best = INT_MAX;
        for (int e = lane; e < E; e += 32) {
          const long long v = S[(g_from * E + e) * G + g_max];
          if (v > best) {
            best = v;
            e_best = e;
          }
        }
        warp_argmax_ll(best, e_best);
        const long long t_move = best;
        if (t_move < q) break;
        long long vmin = (lane < G) ? t : LLONG_MAX;
        int g_min = lane;
        warp_argmin_ll(vmin, g_min);
        if (g_min == g_max || vmin + q > t_avg) break;
        const long long t_s = min(t_move, t_avg - vmin);
        if (lane == 0) {
          S[(g_from * E + e_best) * G + g_max] -= (int)t_s;
          S[(g_from * E + e_best) * G + g_min] += (int)t_s;
          F[g_from * 32 + g_max] -= t_s;
          F[g_from * 32 + g_min] += t_s;
        }
        if (lane == g_max) t -= t_s;
        if (lane == g_min) t += t_s;
        __syncwarp();
        ++iters;
      }
    }
    if (lane == 0 && iters_out != nullptr) *iters_out = iters;
    if (loads_out != nullptr && lane < G) loads_out[lane] = (int)t;
  }
  __syncthreads();
  HM_PSTAMP(3);
}

// ------------------------------------------------------------------------------------------
// layout
// ------------------------------------------------------------------------------------------
// exclusive scan of v[0..n) in place by one warp; returns the total
__device__ int warp_exclusive_scan(int* v, int n, int lane) {
  int running = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int x = (i < n) ? v[i] : 0;
    int incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (i < n) v[i] = running + incl - x;
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
  return running;
}

// block-wide exclusive scan of cnt[0..n) -> out[0..n], out[n] = total
__device__ void block_scan_to(const int* cnt, int n, int* out, int* s_tmp /*[32]*/) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int local = 0;
  for (int i = lo; i < hi; ++i) local += cnt[i];
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_tmp[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int nw = nt / 32;
    const int x = lane < nw ? s_tmp[lane] : 0;
    int ii = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ii, off);
      if (lane >= off) ii += y;
    }
    if (lane < nw) s_tmp[lane] = ii - x;
  }
  __syncthreads();
  int run = s_tmp[w] + incl - local;
  for (int i = lo; i < hi; ++i) {
    out[i] = run;
    run += cnt[i];
  }
  if (tid == nt - 1) out[n] = run;
  __syncthreads();
}

// exclusive scan of cnt[0..n) into out[0..n] (out[n] = total) by ONE warp, no block barrier:
// the fast path's last phase (a block-wide scan cost ~2.7k cycles of barriers at ~128 segments)
__device__ void warp_scan_to(const int* cnt, int n, int32_t* out, int lane) {
  int running = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int x = i < n ? cnt[i] : 0;
    int incl = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    if (i < n) out[i] = running + incl - x;
    running += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) out[n] = running;
}

struct LayoutOut {
  int32_t* slot_base;
  int4* segs;
  int32_t* n_seg;
  int32_t* mprefix;
  int32_t* fetch;
  int32_t* n_fetch;
  int cache_slots;  // EP: fetch cache slots (0 = one per fetched expert); fetch i -> slot n_home + i % cache_slots
  // EP_EXPERT, optional (hm_plan_dispatch): this rank's push work list for the expert-ordered
  // dispatch (hm_dispatch_push_ordered).  Item v = p*G + d is the bucket (me -> d) of the expert at
  // position p of destination d's plan order: (expert, first rank c0 among me's assignments to it,
  // rows, first row in d's receive buffer), rows 0 where d has no p-th expert;
  // push_cprefix[v] = sum of 8-row units of items < v; push_ebase[e] = sum_{e'<e} m_all[me][e'].
  int4* push_items;
  int32_t* push_cprefix;
  int32_t* push_ebase;
};

// plan-order sort key (ascending = execution order): residents first, then more tokens,
// then lower expert id (engine.py:233-234); experts without work sort last
__device__ __forceinline__ unsigned long long plan_key(bool resident, int n, int e) {
  if (n <= 0) return ~0ull;
  return ((unsigned long long)(resident ? 0 : 1) << 62) | ((unsigned long long)(0x7fffffff - n) << 20) |
         (unsigned long long)e;
}

// number of keys[0..n) below `key`, one warp
__device__ __forceinline__ int warp_rank(const unsigned long long* keys, int n, unsigned long long key, int lane) {
  int c = 0;
  for (int j = lane; j < n; j += 32) c += keys[j] < key;
  return (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
}

constexpr int layout_scratch_ints(int G, int E) { return 5 * G * E + 3 + 3 * E + 2; }

// scratch: layout_scratch_ints(G, E) ints (dynamic smem); home: smem copy
__device__ void dev_layout(const int* S, const int* home, int G, int E, int mode, int me, LayoutOut o, int* scratch) {
  __shared__ int s_base[33];
  __shared__ int s_nnz[33];
  __shared__ int s_tmp[32];
  __shared__ int s_scal[4];
  const int GE = G * E;
  int* s_n = scratch;         // LOCAL: n[d][e]; EP: S[g][e][me] as [g][e]
  int* s_off = s_n + GE;      // LOCAL: off[d][e]; EP: recv row of (g,e)
  int* s_cnt = s_off + GE;    // [GE + 1]
  int* s_ne = s_cnt + GE + 1; // [E]
  int* s_nsrc = s_ne + E;     // [E]
  int* s_ord = s_nsrc + E;    // [E]
  // [GE] plan-order keys, 8-byte aligned by pointer arithmetic on the shared array (an integer
  // round trip would drop the shared address space: generic loads in the rank loops)
  unsigned long long* s_key =
      reinterpret_cast<unsigned long long*>(s_ord + E + ((smem_u32(s_ord + E) & 4u) ? 1 : 0));
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nt = blockDim.x;
  HM_PSTAMP(4);

  if (mode == HM_LAYOUT_LOCAL) {
    for (int i = tid; i < GE; i += nt) {
      const int d = i / E, e = i - (i / E) * E;
      int s = 0;
      for (int g = 0; g < G; ++g) s += S[(g * E + e) * G + d];
      s_n[i] = s;
      s_off[i] = s;
    }
    __syncthreads();
    if (w < G) {
      const int total = warp_exclusive_scan(s_off + w * E, E, lane);
      int nz = 0;
      for (int e = lane; e < E; e += 32) nz += (s_n[w * E + e] > 0);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, off);
      if (lane == 0) {
        s_base[w] = total;
        s_nnz[w] = nz;
      }
    }
    __syncthreads();
    if (tid == 0) {
      int run = 0, runz = 0;
      for (int d = 0; d < G; ++d) {
        const int a = s_base[d], z = s_nnz[d];
        s_base[d] = run;
        s_nnz[d] = runz;
        run += a;
        runz += z;
      }
      s_base[G] = run;
      s_nnz[G] = runz;
      *o.n_seg = runz;
      *o.n_fetch = 0;
    }
    __syncthreads();
    if (tid == 0) HM_PHASE(4);
    HM_PSTAMP(5);
    for (int i = tid; i < E * G; i += nt) {
      const int e = i / G, d = i - (i / G) * G;
      int run = s_base[d] + s_off[d * E + e];
      for (int g = 0; g < G; ++g) {
        o.slot_base[(g * E + e) * G + d] = run;
        run += S[(g * E + e) * G + d];
      }
    }
    for (int i = tid; i < GE; i += nt) {
      const int d = i / E, e = i - (i / E) * E;
      s_key[i] = plan_key(home[e] == d, s_n[i], e);
    }
    __syncthreads();
    HM_PSTAMP(6);
    // one thread per (dest, expert): rank = number of smaller plan keys of that dest (the dest's
    // keys are read as shared-memory broadcasts: a warp's 32 entries share d when E >= 32)
    for (int p = tid; p < GE; p += nt) {
      const unsigned long long key = s_key[p];
      if (key == ~0ull) continue;
      const int d = p / E, e = p - d * E;
      const unsigned long long* kd = s_key + d * E;
      int pos = 0;
#pragma unroll 4
      for (int j = 0; j < E; ++j) pos += kd[j] < key;
      const int ne = s_n[p];
      const int sidx = s_nnz[d] + pos;
      o.segs[sidx] = make_int4(s_base[d] + s_off[p], ne, e, e);
      s_cnt[sidx] = (ne + 127) / 128;
    }
    __syncthreads();
    if (tid == 0) HM_PHASE(5);
    HM_PSTAMP(7);
    block_scan_to(s_cnt, s_nnz[G], o.mprefix, s_tmp);
    if (tid == 0) HM_PHASE(6);
    HM_PSTAMP(8);
    return;
  }

  if (mode == HM_LAYOUT_EP_EXPERT) {
    // ---- EP, expert-major receive buffers (one-sided p2p dispatch): rank d's buffer holds rows
    // [expert (ascending id)][source][rank]; every sender derives its rows from the replicated S:
    // slot_base[g,e,d] = sum_{e'<e} n_d(e') + sum_{g'<g} S[g',e,d] (the LOCAL layout with each
    // destination starting at row 0).  Rank me's GEMM work list: ONE segment per expert (all its
    // sources' rows contiguous) in plan order, wslot / fetch list as in HM_LAYOUT_EP.
    for (int i = tid; i < GE; i += nt) {
      const int d = i / E, e = i - (i / E) * E;
      int sum = 0;
      for (int g = 0; g < G; ++g) sum += S[(g * E + e) * G + d];
      s_n[i] = sum;
      s_off[i] = sum;
    }
    __syncthreads();
    HM_PSTAMP(5);
    if (w < G) warp_exclusive_scan(s_off + w * E, E, lane);
    if (tid == 0) {
      s_scal[0] = 0;  // residents with work
      s_scal[1] = 0;  // home experts
      s_scal[2] = 0;  // experts with work
    }
    __syncthreads();
    for (int i = tid; i < E * G; i += nt) {
      const int e = i / G, d = i - (i / G) * G;
      int run = s_off[d * E + e];
      for (int g = 0; g < G; ++g) {
        o.slot_base[(g * E + e) * G + d] = run;
        run += S[(g * E + e) * G + d];
      }
    }
    for (int e = tid; e < E; e += nt) {
      const int ne = s_n[me * E + e];
      const bool re = home[e] == me;
      s_key[e] = plan_key(re, ne, e);
      if (re) atomicAdd(&s_scal[1], 1);
      if (ne > 0) {
        atomicAdd(&s_scal[2], 1);
        if (re) atomicAdd(&s_scal[0], 1);
      }
    }
    __syncthreads();
    HM_PSTAMP(6);
    const int n_res_work = s_scal[0], n_home = s_scal[1], n_work = s_scal[2];
    for (int e = w; e < E; e += nt / 32) {
      const unsigned long long key = s_key[e];
      if (key == ~0ull) continue;  // warp-uniform
      const int oo = warp_rank(s_key, E, key, lane);
      if (lane == 0) {
        int wslot;
        if (home[e] == me) {
          wslot = 0;
          for (int e2 = 0; e2 < e; ++e2) wslot += (home[e2] == me);
        } else {
          const int fi = oo - n_res_work;
          wslot = n_home + (o.cache_slots > 0 ? fi % o.cache_slots : fi);
          o.fetch[fi] = e;
        }
        const int ne = s_n[me * E + e];
        o.segs[oo] = make_int4(s_off[me * E + e], ne, wslot, e);
        s_cnt[oo] = (ne + 127) / 128;
      }
    }
    if (tid == 0) {
      *o.n_seg = n_work;
      *o.n_fetch = n_work - n_res_work;
    }
    __syncthreads();
    HM_PSTAMP(7);
    block_scan_to(s_cnt, n_work, o.mprefix, s_tmp);
    HM_PSTAMP(8);
    return;
  }

  // ---------------- EP mode: this process is rank `me` ----------------
  for (int i = tid; i < GE; i += nt) {
    const int g = i / E, e = i - (i / E) * E;
    const int v = S[(g * E + e) * G + me];
    s_n[i] = v;
    s_off[i] = v;
  }
  __syncthreads();
  if (w < G) {
    const int total = warp_exclusive_scan(s_off + w * E, E, lane);  // within-chunk offsets of source w
    if (lane == 0) s_base[w] = total;                               // flows[w][me]
  }
  __syncthreads();
  if (tid == 0) {
    int run = 0;
    for (int g = 0; g < G; ++g) {
      const int a = s_base[g];
      s_base[g] = run;
      run += a;
    }
    s_base[G] = run;
    s_scal[0] = 0;  // residents with work
    s_scal[1] = 0;  // home experts
    s_scal[2] = 0;  // experts with work
  }
  __syncthreads();
  // send side: slot_base[me,e,d] = send_off[d] + sum_{e'<e} S[me,e',d]  (dest-major send buffer)
  if (w < G) {
    const int d = w;
    int send_off = 0;
    for (int d2 = 0; d2 < d; ++d2)
      for (int e = lane; e < E; e += 32) send_off += S[(me * E + e) * G + d2];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) send_off += __shfl_xor_sync(0xffffffffu, send_off, off);
    int running = send_off;
    for (int base = 0; base < E; base += 32) {
      const int e = base + lane;
      const int x = (e < E) ? S[(me * E + e) * G + d] : 0;
      int incl = x;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      if (e < E) o.slot_base[(me * E + e) * G + d] = running + incl - x;
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  for (int e = tid; e < E; e += nt) {
    int ne = 0, ns = 0;
    for (int g = 0; g < G; ++g) {
      const int v = s_n[g * E + e];
      ne += v;
      ns += (v > 0);
    }
    s_ne[e] = ne;
    s_nsrc[e] = ns;
    s_key[e] = plan_key(home[e] == me, ne, e);
    const bool re = home[e] == me;
    if (re) atomicAdd(&s_scal[1], 1);
    if (ne > 0) {
      atomicAdd(&s_scal[2], 1);
      if (re) atomicAdd(&s_scal[0], 1);
    }
  }
  __syncthreads();
  // one warp per expert: position in the plan order
  for (int e = w; e < E; e += nt / 32) {
    const unsigned long long key = s_key[e];
    if (key == ~0ull) {
      if (lane == 0) s_ord[e] = -1;
      continue;
    }
    const int pos = warp_rank(s_key, E, key, lane);
    if (lane == 0) {
      s_ord[e] = pos;
      s_cnt[pos] = s_nsrc[e];
    }
  }
  __syncthreads();
  const int n_work = s_scal[2];
  if (tid == 0) {
    int run = 0;
    for (int oo = 0; oo < n_work; ++oo) {
      const int a = s_cnt[oo];
      s_cnt[oo] = run;
      run += a;
    }
    s_scal[3] = run;  // number of segments
    *o.n_seg = run;
    *o.n_fetch = n_work - s_scal[0];
  }
  __syncthreads();
  const int n_res_work = s_scal[0];
  const int n_home = s_scal[1];
  for (int e = tid; e < E; e += nt) {
    const int oo = s_ord[e];
    if (oo < 0) continue;
    int wslot;
    if (home[e] == me) {
      wslot = 0;
      for (int e2 = 0; e2 < e; ++e2) wslot += (home[e2] == me);
    } else {
      // bounded cache: fetch i reuses the slot of fetch i - cache_slots, the one whose occupant
      // finishes first (fetched experts compute in plan order; engine.py:239-257)
      const int fi = oo - n_res_work;
      wslot = n_home + (o.cache_slots > 0 ? fi % o.cache_slots : fi);
      o.fetch[fi] = e;
    }
    int sidx = s_cnt[oo];
    for (int g = 0; g < G; ++g) {
      const int v = s_n[g * E + e];
      if (v > 0) {
        o.segs[sidx] = make_int4(s_base[g] + s_off[g * E + e], v, wslot, e);
        ++sidx;
      }
    }
  }
  __syncthreads();
  // per-segment m-tile counts (s_off reused), then scan
  const int n_seg = s_scal[3];
  for (int i = tid; i < n_seg; i += nt) s_off[i] = (o.segs[i].y + 127) / 128;
  __syncthreads();
  block_scan_to(s_off, n_seg, o.mprefix, s_tmp);
}

// ------------------------------------------------------------------------------------------
// fast planner path (plan_kernel): every count < 2^21, policy harmony / none, LOCAL or EP_EXPERT
// layout.  S is kept only transposed, St[g][d][e] (experts on consecutive words), built straight
// from m_all and home; flows and loads are 32-bit.  Same decisions and outputs as dev_schedule +
// dev_layout (bit-exact on the same fixtures): measured with clock64 stamps, the S[g][e][d]
// reads of the general path (G-way bank conflicts: lanes stride G words), its S zero-fill and the
// per-expert serial home-slot count were most of the planner's time.
// ------------------------------------------------------------------------------------------
// rebalance on St / F32 (F32[g*32+d] = sum_e St[g][d][e]); kNch = E/32 chunks per lane, 0 = any E
template <int kNch>
__device__ int rebalance_t(int* St, int* F, int G, int E, int Ep, int q, int lane, int& t_lane, int t_avg) {
  int t = t_lane;
  int iters = 0;
  for (;;) {
    if (__ballot_sync(0xffffffffu, lane < G && t > t_avg) == 0u) break;
    // argmin t does not depend on the rest of the iteration: reduce it alongside argmax t
    const unsigned kmin = __reduce_min_sync(0xffffffffu, lane < G ? ((unsigned)t << 5) | lane : 0xffffffffu);
    const unsigned kmax = __reduce_max_sync(0xffffffffu, lane < G ? ((unsigned)t << 5) | (31u - lane) : 0u);
    const int g_max = 31 - (int)(kmax & 31u);
    const unsigned kf =
        __reduce_max_sync(0xffffffffu, lane < G ? ((unsigned)F[lane * 32 + g_max] << 5) | (31u - lane) : 0u);
    const int g_from = 31 - (int)(kf & 31u);
    const int* col = St + (g_from * G + g_max) * Ep;
    unsigned kb = 0u;
    if (kNch > 0) {
#pragma unroll
      for (int c = 0; c < kNch; ++c) {
        const int e = c * 32 + lane;
        kb = max(kb, ((unsigned)col[e] << 10) | (1023u - e));
      }
    } else {
      for (int e = lane; e < E; e += 32) kb = max(kb, ((unsigned)col[e] << 10) | (1023u - e));
    }
    kb = __reduce_max_sync(0xffffffffu, kb);
    const int t_move = (int)(kb >> 10);
    const int e_max = 1023 - (int)(kb & 1023u);
    if (t_move < q) break;
    const int g_min = (int)(kmin & 31u);
    const int vmin = (int)(kmin >> 5);
    if (g_min == g_max || (long long)vmin + q > t_avg) break;
    const int t_s = min(t_move, t_avg - vmin);
    if (lane == 0) {
      St[(g_from * G + g_max) * Ep + e_max] -= t_s;
      St[(g_from * G + g_min) * Ep + e_max] += t_s;
      F[g_from * 32 + g_max] -= t_s;
      F[g_from * 32 + g_min] += t_s;
    }
    if (lane == g_max) t -= t_s;
    if (lane == g_min) t += t_s;
    __syncwarp();
    ++iters;
  }
  t_lane = t;
  return iters;
}

// Thread mapping of the fast path's per-(dest, expert) passes: G is a power of two dividing the
// block, so thread t owns dest d = t % G for the whole kernel and strides the experts by
// blockDim / G - no integer divisions, [g][e][d]-ordered global stores are coalesced, and with
// every [.][e] row padded to Ep = E + 32/G words a warp's (e, d) reads hit 32 distinct banks.
struct DestLanes {
  int d, e0, step;
};
__device__ __forceinline__ DestLanes dest_lanes(int G) {
  const int lg = 31 - __clz(G);
  return DestLanes{(int)(threadIdx.x & (G - 1)), (int)(threadIdx.x >> lg), (int)(blockDim.x >> lg)};
}

// initial_assign + rebalance into St[g][d][e] (rows of Ep words); S_out[g][e][d] written from St
__device__ void dev_schedule_t(int* St, int Ep, int* F, const int* m, const int* home, int G, int E, int q,
                               int rebalance, int32_t* __restrict__ S_out, int32_t* iters_out, int32_t* loads_out) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  // initial_assign (policies.py:109-117): bucket (g, e) starts on home[e]; flows F[g][d] on the fly
  for (int row = w; row < G * G; row += nw) {
    const int g = row >> (31 - __clz(G)), d = row & (G - 1);
    int f = 0;
    for (int e = lane; e < E; e += 32) {
      const int v = (home[e] == d) ? m[g * E + e] : 0;
      St[row * Ep + e] = v;
      f += v;
    }
    f = (int)__reduce_add_sync(0xffffffffu, (unsigned)f);
    if (lane == 0) F[g * 32 + d] = f;
  }
  __syncthreads();
  HM_PSTAMP(2);
  if (w == 0) {
    int t = 0;
    if (lane < G)
      for (int g = 0; g < G; ++g) t += F[g * 32 + lane];
    const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)t);  // lanes >= G hold 0
    const int t_avg = total / G;
    int iters = 0;
    if (rebalance == HM_POLICY_REBALANCE) {
      if (E == 128)
        iters = rebalance_t<4>(St, F, G, E, Ep, q, lane, t, t_avg);
      else if (E == 64)
        iters = rebalance_t<2>(St, F, G, E, Ep, q, lane, t, t_avg);
      else if (E == 256)
        iters = rebalance_t<8>(St, F, G, E, Ep, q, lane, t, t_avg);
      else
        iters = rebalance_t<0>(St, F, G, E, Ep, q, lane, t, t_avg);
    }
    if (lane == 0 && iters_out != nullptr) *iters_out = iters;
    if (loads_out != nullptr && lane < G) loads_out[lane] = t;
  }
  __syncthreads();
  HM_PSTAMP(3);
  const DestLanes L = dest_lanes(G);
  for (int g = 0; g < G; ++g) {
    const int* row = St + (g * G + L.d) * Ep;
    for (int e = L.e0; e < E; e += L.step) S_out[(g * E + e) * G + L.d] = row[e];
  }
}

// plan-order key in 32 bits (counts < 2^21, E <= 1024): residents first, then more tokens, then
// lower expert id (engine.py:233-234); experts without work sort last.  Same order as plan_key.
__device__ __forceinline__ unsigned plan_key32(bool resident, int n, int e) {
  if (n <= 0) return 0xffffffffu;
  return ((resident ? 0u : 1u) << 31) | ((unsigned)((1 << 21) - 1 - n) << 10) | (unsigned)e;
}

// fast-path layout scratch (ints): s_n, s_off [G][Ep], s_cnt [G*E + 1], s_key [G][Ep] (+3 for
// 16-byte alignment), s_hr [E]
constexpr int fast_layout_scratch_ints(int G, int E) { return 3 * G * (E + 32 / G) + 2 * (G * E + 1) + 3 + E; }
constexpr int plan_scratch_ints(int G, int E) {
  return layout_scratch_ints(G, E) > fast_layout_scratch_ints(G, E) ? layout_scratch_ints(G, E)
                                                                     : fast_layout_scratch_ints(G, E);
}

// LOCAL / EP_EXPERT layouts from St (same outputs as dev_layout)
__device__ void dev_layout_t(const int* St, int Ep, const int* home, int G, int E, int mode, int me, LayoutOut o,
                             int* scratch) {
  __shared__ int s_base[33];
  __shared__ int s_nnz[33];
  __shared__ int s_tmp[32];
  __shared__ int s_scal[4];
  const int GE = G * E;
  int* s_n = scratch;            // n[d][e] = rows of expert e on dest d (rows of Ep)
  int* s_off = s_n + G * Ep;     // exclusive scan of n[d][.] over experts (rows of Ep)
  int* s_cnt = s_off + G * Ep;   // [GE + 1] 128-row tiles per segment (plan order)
  // [G][Ep] plan-order keys, 16-byte aligned for the vector rank loads (pointer arithmetic on the
  // shared array keeps the shared address space)
  int* key_base = s_cnt + GE + 1;
  unsigned* s_key = reinterpret_cast<unsigned*>(key_base + ((4u - ((smem_u32(key_base) >> 2) & 3u)) & 3u));
  int* s_hr = reinterpret_cast<int*>(s_key + G * Ep);  // [E] EP: home-slot rank
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const DestLanes L = dest_lanes(G);
  const bool local = mode == HM_LAYOUT_LOCAL;
  HM_PSTAMP(4);
  for (int e = L.e0; e < E; e += L.step) {
    int sum = 0;
    for (int g = 0; g < G; ++g) sum += St[(g * G + L.d) * Ep + e];
    s_n[L.d * Ep + e] = sum;
    s_off[L.d * Ep + e] = sum;
    if (local) s_key[L.d * Ep + e] = plan_key32(home[e] == L.d, sum, e);
  }
  if (!local) {  // home-slot rank of every expert: ballots over warp chunks
    for (int e0 = 0; e0 < E; e0 += blockDim.x) {
      const int e = e0 + tid;
      const bool mine = e < E && home[e] == me;
      const unsigned mask = __ballot_sync(0xffffffffu, mine);
      if (lane == 0) s_tmp[w] = __popc(mask);
      __syncthreads();
      if (e < E) {
        int r = e0 > 0 ? s_hr[e0 - 1] + (home[e0 - 1] == me) : 0;
        for (int w2 = 0; w2 < w; ++w2) r += s_tmp[w2];
        s_hr[e] = r + __popc(mask & ((1u << lane) - 1u));
      }
      __syncthreads();
    }
  }
  __syncthreads();
  HM_PSTAMP(5);
  if (w < G) {
    const int total = warp_exclusive_scan(s_off + w * Ep, E, lane);
    int nz = 0;
    for (int e = lane; e < E; e += 32) nz += (s_n[w * Ep + e] > 0);
    nz = (int)__reduce_add_sync(0xffffffffu, (unsigned)nz);
    if (lane == 0) {
      s_base[w] = total;
      s_nnz[w] = nz;
    }
  }
  if (tid == 0) {
    s_scal[0] = 0;  // residents with work (EP)
    s_scal[1] = 0;  // home experts (EP)
    s_scal[2] = 0;  // experts with work (EP)
  }
  if (!local) {
    for (int e = tid; e < E; e += blockDim.x) s_key[e] = plan_key32(home[e] == me, s_n[me * Ep + e], e);
  }
  __syncthreads();
  if (local && tid == 0) {
    int run = 0, runz = 0;
    for (int d = 0; d < G; ++d) {
      const int a = s_base[d], z = s_nnz[d];
      s_base[d] = run;
      s_nnz[d] = runz;
      run += a;
      runz += z;
    }
    s_base[G] = run;
    s_nnz[G] = runz;
    *o.n_seg = runz;
    *o.n_fetch = 0;
  }
  if (!local) {
    for (int e = tid; e < E; e += blockDim.x) {
      const bool re = home[e] == me;
      if (re) atomicAdd(&s_scal[1], 1);
      if (s_n[me * Ep + e] > 0) {
        atomicAdd(&s_scal[2], 1);
        if (re) atomicAdd(&s_scal[0], 1);
      }
    }
  }
  __syncthreads();
  // slot_base[g,e,d] = base(d) + off[d][e] + sum_{g'<g} S[g',e,d] (EP_EXPERT: base(d) = 0)
  for (int e = L.e0; e < E; e += L.step) {
    int run = (local ? s_base[L.d] : 0) + s_off[L.d * Ep + e];
    for (int g = 0; g < G; ++g) {
      o.slot_base[(g * E + e) * G + L.d] = run;
      run += St[(g * G + L.d) * Ep + e];
    }
  }
  HM_PSTAMP(6);
  if (local) {
    // one thread per (dest, expert): rank among the dest's keys (keys are distinct: the expert id
    // is part of the key); 128-bit loads of the dest's key row
    const bool vec = ((E | Ep) & 3) == 0;
    for (int e = L.e0; e < E; e += L.step) {
      const int d = L.d;
      const unsigned key = s_key[d * Ep + e];
      if (key == 0xffffffffu) continue;
      const unsigned* kd = s_key + d * Ep;
      int pos = 0;
      if (vec) {
        const uint4* kd4 = reinterpret_cast<const uint4*>(kd);
#pragma unroll 4
        for (int j = 0; j < E / 4; ++j) {
          const uint4 v = kd4[j];
          pos += (v.x < key) + (v.y < key) + (v.z < key) + (v.w < key);
        }
      } else {
        for (int j = 0; j < E; ++j) pos += kd[j] < key;
      }
      const int ne = s_n[d * Ep + e];
      const int sidx = s_nnz[d] + pos;
      o.segs[sidx] = make_int4(s_base[d] + s_off[d * Ep + e], ne, e, e);
      s_cnt[sidx] = (ne + 127) / 128;
    }
    __syncthreads();
    HM_PSTAMP(7);
    if (w == 0) warp_scan_to(s_cnt, s_nnz[G], o.mprefix, lane);
    HM_PSTAMP(8);
    return;
  }
  const int n_res_work = s_scal[0], n_home = s_scal[1], n_work = s_scal[2];
  for (int e = tid; e < E; e += blockDim.x) {
    const unsigned key = s_key[e];
    if (key == 0xffffffffu) continue;
    int oo = 0;
    for (int j = 0; j < E; ++j) oo += s_key[j] < key;
    int wslot;
    if (home[e] == me) {
      wslot = s_hr[e];
    } else {
      // bounded cache: fetch i reuses the slot of fetch i - cache_slots, the one whose occupant
      // finishes first (fetched experts compute in plan order; engine.py:239-257)
      const int fi = oo - n_res_work;
      wslot = n_home + (o.cache_slots > 0 ? fi % o.cache_slots : fi);
      o.fetch[fi] = e;
    }
    const int ne = s_n[me * Ep + e];
    o.segs[oo] = make_int4(s_off[me * Ep + e], ne, wslot, e);
    s_cnt[oo] = (ne + 127) / 128;
  }
  if (tid == 0) {
    *o.n_seg = n_work;
    *o.n_fetch = n_work - n_res_work;
  }
  __syncthreads();
  HM_PSTAMP(7);
  if (w == 0) warp_scan_to(s_cnt, n_work, o.mprefix, lane);
  if (o.push_items != nullptr) {
    // push work list for the expert-ordered dispatch: every destination's plan order (keys of
    // all (d, e); s_key is free again), this rank's bucket of each (position, destination)
    int* s_pc = s_hr + E;  // [GE + 1] 8-row push units per item
    for (int e = L.e0; e < E; e += L.step) s_key[L.d * Ep + e] = plan_key32(home[e] == L.d, s_n[L.d * Ep + e], e);
    for (int v = tid; v < GE; v += blockDim.x) {
      o.push_items[v] = make_int4(0, 0, 0, 0);
      s_pc[v] = 0;
    }
    __syncthreads();
    const bool vec = ((E | Ep) & 3) == 0;
    for (int e = L.e0; e < E; e += L.step) {
      const int d = L.d;
      const unsigned key = s_key[d * Ep + e];
      if (key == 0xffffffffu) continue;
      const unsigned* kd = s_key + d * Ep;
      int pos = 0;
      if (vec) {
        const uint4* kd4 = reinterpret_cast<const uint4*>(kd);
#pragma unroll 4
        for (int j = 0; j < E / 4; ++j) {
          const uint4 v = kd4[j];
          pos += (v.x < key) + (v.y < key) + (v.z < key) + (v.w < key);
        }
      } else {
        for (int j = 0; j < E; ++j) pos += kd[j] < key;
      }
      const int cnt = St[(me * G + d) * Ep + e];
      int c0 = 0;
      for (int d2 = 0; d2 < d; ++d2) c0 += St[(me * G + d2) * Ep + e];
      int row0 = s_off[d * Ep + e];
      for (int g = 0; g < me; ++g) row0 += St[(g * G + d) * Ep + e];
      o.push_items[pos * G + d] = make_int4(e, c0, cnt, row0);
      s_pc[pos * G + d] = (cnt + 7) >> 3;  // 8-row push units (hm_dispatch_push_ordered)
    }
    __syncthreads();
    block_scan_to(s_pc, GE, o.push_cprefix, s_tmp);
    if (w == 0) {  // ebase: exclusive scan of this rank's histogram row m_all[me][.]
      int running = 0;
      for (int base = 0; base < E; base += 32) {
        const int e = base + lane;
        int x = 0;
        if (e < E)
          for (int d = 0; d < G; ++d) x += St[(me * G + d) * Ep + e];
        int incl = x;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += y;
        }
        if (e < E) o.push_ebase[e] = running + incl - x;
        running += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) o.push_ebase[E] = running;
    }
  }
  HM_PSTAMP(8);
}

// ------------------------------------------------------------------------------------------
// kernels
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) hist_scan_kernel(const int32_t* __restrict__ tile_hist, int n_ranks, int tpr,
                                                         int E,
                                 int32_t* __restrict__ hist, int32_t* __restrict__ tile_off) {
  __shared__ int s_part[8 * 128];
  dev_hist_reduce(tile_hist, n_ranks, tpr, E, hist, nullptr, tile_off, s_part);
}

template <bool kSmemS, bool kFromS>
__global__ void __launch_bounds__(256)
    schedule_kernel(const int32_t* __restrict__ m_all, const int32_t* __restrict__ home, int G, int E, int q,
                    int rebalance, int32_t* __restrict__ S_out, int32_t* __restrict__ iters_out,
                    int32_t* __restrict__ loads_out) {
  extern __shared__ int s_dyn[];
  __shared__ long long F[32 * 32];
  const int n = G * E * G;
  // batched launches: CTA b schedules instance b (a layer of a trace, ...)
  const int b = blockIdx.x;
  if (m_all != nullptr) m_all += (int64_t)b * G * E;
  S_out += (int64_t)b * n;
  iters_out += b;
  if (loads_out != nullptr) loads_out += (int64_t)b * G;
  int* S = kSmemS ? s_dyn : S_out;
  if (kFromS && kSmemS)
    for (int i = threadIdx.x; i < n; i += blockDim.x) S[i] = S_out[i];
  dev_schedule(S, !kFromS, m_all, home, G, E, q, rebalance, iters_out, loads_out, F, kSmemS ? s_dyn + n : nullptr);
  if (kSmemS)
    for (int i = threadIdx.x; i < n; i += blockDim.x) S_out[i] = S[i];
}

__global__ void __launch_bounds__(kPlanThreads)
    layout_kernel(const int32_t* __restrict__ S, const int32_t* __restrict__ home, int G, int E, int mode, int me,
                  LayoutOut o) {
  extern __shared__ int s_lay[];
  dev_layout(S, home, G, E, mode, me, o, s_lay);
}

// Single-GPU planner (G = 1, LOCAL): nothing can move, so the schedule is S = m and the layout
// reduces to one scan and one sort of the experts - done with one thread per expert instead of
// the general (dest, expert) machinery.  Outputs are identical to plan_kernel<true> at G = 1:
// rows expert-major, segments in plan order (all experts resident: more tokens first, then
// lower id, engine.py:233-234), no fetches.
__global__ void __launch_bounds__(kPlanThreads)
    plan_g1_kernel(const int32_t* __restrict__ tile_hist, int tpr, int E, int32_t* __restrict__ m_out,
                   int32_t* __restrict__ tile_off, int32_t* __restrict__ S_out, int32_t* __restrict__ iters_out,
                   int32_t* __restrict__ loads_out, LayoutOut o) {
  extern __shared__ int s_dyn[];
  __shared__ int s_part[8 * 128];
  int* s_m = s_dyn;                 // [E]
  int* s_base = s_m + E;            // [E + 1] expert-major row starts
  int* s_cnt = s_base + E + 1;      // [E + 1] 128-row tiles per segment, plan order
  unsigned long long* s_key =       // [E] plan-order keys (8-byte aligned, shared address space kept)
      reinterpret_cast<unsigned long long*>(s_cnt + E + 1 + ((smem_u32(s_cnt + E + 1) & 4u) ? 1 : 0));
  const int tid = threadIdx.x;
  if (tid == 0) HM_PHASE(0);
  dev_hist_reduce(tile_hist, 1, tpr, E, s_m, m_out, tile_off, s_part);
  if (tid == 0) HM_PHASE(1);
  for (int e = tid; e < E; e += blockDim.x) {
    const int n = s_m[e];
    S_out[e] = n;  // S[0, e, 0]
    s_key[e] = plan_key(true, n, e);
  }
  // s_base = exclusive scan of the counts (s_base[E] = total): one warp, then the block barrier
  // that also publishes the keys
  if ((tid >> 5) == 0) warp_scan_to(s_m, E, s_base, tid & 31);
  __syncthreads();
  if (tid == 0) {
    HM_PHASE(2);
    *iters_out = 0;
    if (loads_out != nullptr) loads_out[0] = s_base[E];
    *o.n_fetch = 0;
  }
  int nseg = 0;
  for (int e0 = 0; e0 < E; e0 += blockDim.x) {
    const int e = e0 + tid;
    const unsigned long long key = e < E ? s_key[e] : ~0ull;
    if (key != ~0ull) {
      int rank = 0;  // keys are distinct (the expert id is part of the key)
      for (int j = 0; j < E; ++j) rank += s_key[j] < key;
      const int n = s_m[e];
      o.segs[rank] = make_int4(s_base[e], n, e, e);
      s_cnt[rank] = (n + 127) / 128;
    }
    if (e < E) o.slot_base[e] = s_base[e];
    nseg += __syncthreads_count(key != ~0ull);
  }
  if (tid == 0) *o.n_seg = nseg;
  if ((tid >> 5) == 0) warp_scan_to(s_cnt, nseg, o.mprefix, tid & 31);
  if (tid == 0) HM_PHASE(3);
}

// Whole planning stage in one launch.  kHist: m_all comes from the router's tile
// histograms (LOCAL, n_ranks = G); otherwise from m_in (EP: the all-gathered m_all).
template <bool kHist>
__global__ void __launch_bounds__(kPlanThreads)
    plan_kernel(const int32_t* __restrict__ tile_hist, int tpr, const int32_t* __restrict__ m_in,
                const int32_t* __restrict__ home_g, int G, int E, int q, int rebalance, int mode, int me,
                int32_t* __restrict__ m_out, int32_t* __restrict__ tile_off, int32_t* __restrict__ S_out,
                int32_t* __restrict__ iters_out, int32_t* __restrict__ loads_out, LayoutOut o, int fast) {
  extern __shared__ int s_dyn[];
  __shared__ long long F[32 * 32];
  __shared__ int s_part[8 * 128];
  const int GE = G * E;
  int* s_home = s_dyn;            // [E]
  int* s_m = s_home + E;          // [G*E]
  int* s_S = s_m + GE;            // [G*E*G]
  int* s_scr = s_S + GE * G;      // layout scratch [3*G*E + 1 + 3*E]
  int* s_St = s_scr + plan_scratch_ints(G, E);  // [G*G*E] transposed S (fast path: [G*G][E + 32/G])
#ifdef HM_PLAN_TWICE  // diagnostics: run the whole plan twice, the stamps keep the second (warm icache) pass
  for (int rep = 0; rep < 2; ++rep) {
  __syncthreads();
#endif
  if (threadIdx.x == 0) HM_PHASE(0);
  HM_PSTAMP(0);
#ifdef HM_PLAN_CLOCK
  const long long c0 = clock64();
#endif
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_home[i] = home_g[i];
  if (kHist) {
    dev_hist_reduce(tile_hist, G, tpr, E, s_m, m_out, tile_off, s_part);
  } else {
    for (int i = threadIdx.x; i < GE; i += blockDim.x) s_m[i] = m_in[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) HM_PHASE(1);
  HM_PSTAMP(1);
  // fast path: every count < 2^21 (32-bit packed keys), harmony / static policy, LOCAL or
  // EP_EXPERT layout (HM_PLAN_FAST=0 forces the general path: A/B and tests)
  __shared__ unsigned long long s_wpart[32];  // per-warp partial sums of m_all (one barrier, no atomics)
  {
    unsigned long long part = 0ull;
    for (int i = threadIdx.x; i < GE; i += blockDim.x) part += (unsigned)s_m[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if ((threadIdx.x & 31) == 0) s_wpart[threadIdx.x >> 5] = part;
  }
  __syncthreads();
  unsigned long long s_total = 0ull;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s_total += s_wpart[w];
  if (fast && s_total < (1ull << 21) && rebalance != HM_POLICY_EVEN_SPLIT && mode != HM_LAYOUT_EP &&
      (G & (G - 1)) == 0) {
    const int Ep = E + 32 / G;
    dev_schedule_t(s_St, Ep, reinterpret_cast<int*>(F), s_m, s_home, G, E, q, rebalance, S_out, iters_out,
                   loads_out);
    if (threadIdx.x == 0) HM_PHASE(2);
    dev_layout_t(s_St, Ep, s_home, G, E, mode, me, o, s_scr);
  } else {
    // the push work list exists only on the fast path: flag it invalid (the push kernel traps)
    if (o.push_cprefix != nullptr && threadIdx.x == 0) o.push_cprefix[GE] = -1;
    dev_schedule(s_S, true, s_m, s_home, G, E, q, rebalance, iters_out, loads_out, F, s_St);
    if (threadIdx.x == 0) HM_PHASE(2);
    for (int i = threadIdx.x; i < GE * G; i += blockDim.x) S_out[i] = s_S[i];
    dev_layout(s_S, s_home, G, E, mode, me, o, s_scr);
  }
  if (threadIdx.x == 0) HM_PHASE(3);
#ifdef HM_PLAN_CLOCK
  if (threadIdx.x == 0) g_phase_ns[7] = (unsigned long long)(clock64() - c0);
#endif
#ifdef HM_PLAN_TWICE
  }
#endif
}

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------
int launch_hist_scan(const int32_t* tile_hist, int n_ranks, int tiles_per_rank, int E, int32_t* hist,
                     int32_t* tile_off, cudaStream_t stream) {
  if (n_ranks < 1 || tiles_per_rank < 0 || E < 1) return set_error(HM_EINVAL, "hist_scan: bad sizes");
  hist_scan_kernel<<<1, 1024, 0, stream>>>(tile_hist, n_ranks, tiles_per_rank, E, hist, tile_off);
  return check_launch("hist_scan");
}

int launch_schedule_batched(const int32_t* m_all, const int32_t* home, int B, int G, int E, int q, int rebalance,
                            int32_t* S, int32_t* iters, int32_t* loads, cudaStream_t stream) {
  if (q < 1) return set_error(HM_EINVAL, "token threshold q must be >= 1");
  if (G < 1 || G > 32 || E < 1) return set_error(HM_EINVAL, "schedule: need 1 <= G <= 32 and E >= 1");
  if (rebalance < HM_POLICY_NONE || rebalance > HM_POLICY_EVEN_SPLIT)
    return set_error(HM_EINVAL, "schedule: unknown policy code");
  if (B < 0) return set_error(HM_EINVAL, "schedule: batch count must be >= 0");
  if (B == 0) return HM_OK;
  const size_t sbytes = (size_t)2 * G * E * G * sizeof(int);  // S + transposed copy for the fast loop
  if (sbytes <= 200 * 1024) {
    cudaFuncSetAttribute(schedule_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes);
    schedule_kernel<true, false><<<B, 256, sbytes, stream>>>(m_all, home, G, E, q, rebalance, S, iters, loads);
  } else {
    schedule_kernel<false, false><<<B, 256, 0, stream>>>(m_all, home, G, E, q, rebalance, S, iters, loads);
  }
  return check_launch("schedule");
}

int launch_schedule(const int32_t* m_all, const int32_t* home, int G, int E, int q, int rebalance, int32_t* S,
                    int32_t* iters, int32_t* loads, cudaStream_t stream) {
  return launch_schedule_batched(m_all, home, 1, G, E, q, rebalance, S, iters, loads, stream);
}

int launch_rebalance(int32_t* S, int G, int E, int q, int32_t* iters, int32_t* loads, cudaStream_t stream) {
  if (q < 1) return set_error(HM_EINVAL, "token threshold q must be >= 1");
  if (G < 1 || G > 32 || E < 1) return set_error(HM_EINVAL, "rebalance: need 1 <= G <= 32 and E >= 1");
  const size_t sbytes = (size_t)2 * G * E * G * sizeof(int);  // S + transposed copy for the fast loop
  if (sbytes <= 200 * 1024) {
    cudaFuncSetAttribute(schedule_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes);
    schedule_kernel<true, true><<<1, 256, sbytes, stream>>>(nullptr, nullptr, G, E, q, 1, S, iters, loads);
  } else {
    schedule_kernel<false, true><<<1, 256, 0, stream>>>(nullptr, nullptr, G, E, q, 1, S, iters, loads);
  }
  return check_launch("rebalance");
}

static int check_layout_args(int G, int E, int mode, int me) {
  if (G < 1 || G > 32 || E < 1 || E > 1024 || G * E > kLayMaxGE)
    return set_error(HM_EINVAL, "dispatch_layout: need G <= 32, E <= 1024, G*E <= 8192");
  if (mode != HM_LAYOUT_LOCAL && mode != HM_LAYOUT_EP && mode != HM_LAYOUT_EP_EXPERT)
    return set_error(HM_EINVAL, "dispatch_layout: bad mode");
  if (mode != HM_LAYOUT_LOCAL && (me < 0 || me >= G)) return set_error(HM_EINVAL, "dispatch_layout: bad rank");
  return HM_OK;
}

int launch_layout(const int32_t* S, const int32_t* home, int G, int E, int mode, int me, int32_t* slot_base,
                  int32_t* segs, int32_t* n_seg, int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch,
                  int cache_slots, cudaStream_t stream) {
  int rc = check_layout_args(G, E, mode, me);
  if (rc) return rc;
  if (cache_slots < 0) return set_error(HM_EINVAL, "dispatch_layout: cache_slots must be >= 0");
  const size_t smem = (size_t)layout_scratch_ints(G, E) * sizeof(int);
  cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  LayoutOut o{slot_base, reinterpret_cast<int4*>(segs), n_seg, mtile_prefix, fetch, n_fetch, cache_slots};
  layout_kernel<<<1, kPlanThreads, smem, stream>>>(S, home, G, E, mode, me, o);
  return check_launch("dispatch_layout");
}

static bool use_plan_g1() {  // HM_PLAN_G1=0: the general planner at G = 1 too (A/B, tests)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HM_PLAN_G1");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int plan_fast() {  // HM_PLAN_FAST=0: the general (S-layout, 64-bit) planner path everywhere
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HM_PLAN_FAST");
    v = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return v;
}

int launch_plan(const int32_t* tile_hist, int tiles_per_rank, const int32_t* m_in, const int32_t* home, int G, int E,
                int q, int rebalance, int mode, int me, int32_t* m_out, int32_t* tile_off, int32_t* S, int32_t* iters,
                int32_t* loads, int32_t* slot_base, int32_t* segs, int32_t* n_seg, int32_t* mtile_prefix,
                int32_t* fetch, int32_t* n_fetch, int cache_slots, cudaStream_t stream, int32_t* push_items,
                int32_t* push_cprefix, int32_t* push_ebase) {
  if (q < 1) return set_error(HM_EINVAL, "token threshold q must be >= 1");
  if (cache_slots < 0) return set_error(HM_EINVAL, "plan: cache_slots must be >= 0");
  int rc = check_layout_args(G, E, mode, me);
  if (rc) return rc;
  if (rebalance < HM_POLICY_NONE || rebalance > HM_POLICY_EVEN_SPLIT)
    return set_error(HM_EINVAL, "plan: unknown policy code");
  const bool hist = tile_hist != nullptr;
  if (hist && mode != HM_LAYOUT_LOCAL) return set_error(HM_EINVAL, "plan: tile histograms imply the LOCAL layout");
  if (!hist && m_in == nullptr) return set_error(HM_EINVAL, "plan: need tile_hist or m_all");
  const size_t smem = (size_t)(E + G * E + 2 * G * E * G + 32 * G + plan_scratch_ints(G, E)) * sizeof(int);
  if (smem > 200 * 1024) return set_error(HM_EINVAL, "plan: G*E*G too large for the fused planner; use hm_schedule");
  if (push_items != nullptr) {
    if (mode != HM_LAYOUT_EP_EXPERT || push_cprefix == nullptr || push_ebase == nullptr)
      return set_error(HM_EINVAL, "plan: the push work list needs the EP_EXPERT layout, cprefix and ebase");
    if ((G & (G - 1)) != 0 || rebalance == HM_POLICY_EVEN_SPLIT || !plan_fast())
      return set_error(HM_EINVAL, "plan: the push work list needs a power-of-two G and the fast planner path");
  }
  LayoutOut o{slot_base,   reinterpret_cast<int4*>(segs), n_seg, mtile_prefix, fetch, n_fetch, cache_slots,
              reinterpret_cast<int4*>(push_items), push_cprefix, push_ebase};
  if (hist && G == 1 && use_plan_g1()) {
    const size_t smem1 = (size_t)(3 * E + 2) * sizeof(int) + 8 + (size_t)E * 8;
    cudaFuncSetAttribute(plan_g1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    plan_g1_kernel<<<1, kPlanThreads, smem1, stream>>>(tile_hist, tiles_per_rank, E, m_out, tile_off, S, iters, loads,
                                                       o);
  } else if (hist) {
    cudaFuncSetAttribute(plan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    plan_kernel<true><<<1, kPlanThreads, smem, stream>>>(tile_hist, tiles_per_rank, nullptr, home, G, E, q, rebalance,
                                                         mode, me, m_out, tile_off, S, iters, loads, o, plan_fast());
  } else {
    cudaFuncSetAttribute(plan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    plan_kernel<false><<<1, kPlanThreads, smem, stream>>>(nullptr, 0, m_in, home, G, E, q, rebalance, mode, me,
                                                          m_out, tile_off, S, iters, loads, o, plan_fast());
  }
  return check_launch("plan");
}

}  // namespace hm
