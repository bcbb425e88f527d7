// K3: HarMoEny scheduler on the GPU, plus the dispatch/GEMM layout it implies.
//
// schedule_kernel restates moesim/policies.py:109-141 (initial_assign +
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
// layout_kernel turns S into (a) slot_base[g,e,d], the buffer row of the first
// token of every bucket, and (b) the grouped GEMM's segment list in the
// per-GPU execution order of plan_gpu_execution (engine.py:233-234: resident
// experts with work by (-tokens, e), then fetched experts by (-tokens, e)).
#include <climits>

#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

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

template <bool kSmemS, bool kFromS>
__global__ void __launch_bounds__(256)
    schedule_kernel(const int32_t* __restrict__ m_all, const int32_t* __restrict__ home, int G, int E, int q,
                    int rebalance, int32_t* __restrict__ S_out, int32_t* __restrict__ iters_out,
                    int32_t* __restrict__ loads_out) {
  extern __shared__ int s_dyn[];
  __shared__ long long F[32 * 32];
  int* S = kSmemS ? s_dyn : S_out;
  const int n = G * E * G;
  if (kFromS) {
    // rebalance an arbitrary schedule in place (policies.py:144-171)
    if (kSmemS)
      for (int i = threadIdx.x; i < n; i += blockDim.x) S[i] = S_out[i];
  } else {
    // initial_assign (policies.py:109-117)
    for (int i = threadIdx.x; i < n; i += blockDim.x) S[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < G * E; i += blockDim.x) {
      const int g = i / E, e = i - (i / E) * E;
      S[(g * E + e) * G + home[e]] = m_all[i];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * G; i += blockDim.x) {
    const int g = i / G, d = i - (i / G) * G;
    long long f = 0;
    for (int e = 0; e < E; ++e) f += S[(g * E + e) * G + d];
    F[g * 32 + d] = f;
  }
  __syncthreads();

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
    if (rebalance) {
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
    if (lane == 0) *iters_out = iters;
    if (loads_out != nullptr && lane < G) loads_out[lane] = (int)t;
  }
  __syncthreads();
  if (kSmemS)
    for (int i = threadIdx.x; i < n; i += blockDim.x) S_out[i] = S[i];
}

// ------------------------------------------------------------------------------------------
// layout
// ------------------------------------------------------------------------------------------
constexpr int kLayThreads = 1024;
constexpr int kLayMaxGE = 8192;  // G*E entries kept in smem

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

// block-wide exclusive scan of cnt[0..n) -> out[0..n], out[n] = total (1024 threads)
__device__ void block_scan_to(const int* cnt, int n, int* out, int* s_tmp /*[32]*/) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = (n + kLayThreads - 1) / kLayThreads;
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
    int x = s_tmp[lane];
    int ii = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, ii, off);
      if (lane >= off) ii += y;
    }
    s_tmp[lane] = ii - x;
  }
  __syncthreads();
  int run = s_tmp[w] + incl - local;
  for (int i = lo; i < hi; ++i) {
    out[i] = run;
    run += cnt[i];
  }
  if (tid == kLayThreads - 1) out[n] = run;
  __syncthreads();
}

// plan order key: residents first, then more tokens first, then lower expert id
__device__ __forceinline__ bool plan_before(bool ra, int na, int a, bool rb, int nb, int b) {
  if (ra != rb) return ra;
  if (na != nb) return na > nb;
  return a < b;
}

__global__ void __launch_bounds__(kLayThreads)
    layout_kernel(const int32_t* __restrict__ S, const int32_t* __restrict__ home, int G, int E, int mode, int me,
                  int32_t* __restrict__ slot_base, int4* __restrict__ segs, int32_t* __restrict__ n_seg_out,
                  int32_t* __restrict__ mprefix, int32_t* __restrict__ fetch, int32_t* __restrict__ n_fetch_out) {
  extern __shared__ int s_lay[];
  const int GE = G * E;
  int* s_n = s_lay;                 // LOCAL: n[d][e]; EP: S[g][e][me] as [g][e]
  int* s_off = s_n + GE;            // LOCAL: off[d][e]; EP: recv row of (g,e)
  int* s_cnt = s_off + GE;          // [GE + 1]
  int* s_ne = s_cnt + GE + 1;       // [E]
  int* s_nsrc = s_ne + E;           // [E]
  int* s_ord = s_nsrc + E;          // [E]
  __shared__ int s_base[33];
  __shared__ int s_nnz[33];
  __shared__ int s_tmp[32];
  __shared__ int s_scal[4];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;

  if (mode == HM_LAYOUT_LOCAL) {
    for (int i = tid; i < G * E; i += kLayThreads) {
      const int d = i / E, e = i - (i / E) * E;
      int s = 0;
      for (int g = 0; g < G; ++g) s += S[(g * E + e) * G + d];
      s_n[i] = s;
      s_off[i] = s;
    }
    __syncthreads();
    // per-destination exclusive scan over experts (warp d) + count of experts with work
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
      *n_seg_out = runz;
      *n_fetch_out = 0;
    }
    __syncthreads();
    // slot_base[g,e,d] = base[d] + off[d][e] + sum_{g'<g} S[g',e,d]
    for (int i = tid; i < E * G; i += kLayThreads) {
      const int e = i / G, d = i - (i / G) * G;
      int run = s_base[d] + s_off[d * E + e];
      for (int g = 0; g < G; ++g) {
        slot_base[(g * E + e) * G + d] = run;
        run += S[(g * E + e) * G + d];
      }
    }
    // segments in plan order per destination
    for (int i = tid; i < G * E; i += kLayThreads) {
      const int d = i / E, e = i - (i / E) * E;
      const int ne = s_n[i];
      if (ne <= 0) continue;
      const bool re = home[e] == d;
      int pos = 0;
      for (int e2 = 0; e2 < E; ++e2) {
        const int n2 = s_n[d * E + e2];
        if (n2 > 0 && plan_before(home[e2] == d, n2, e2, re, ne, e)) ++pos;
      }
      const int sidx = s_nnz[d] + pos;
      segs[sidx] = make_int4(s_base[d] + s_off[i], ne, e, e);
      s_cnt[sidx] = (ne + 127) / 128;
    }
    __syncthreads();
    block_scan_to(s_cnt, s_nnz[G], mprefix, s_tmp);
    return;
  }

  // ---------------- EP mode: this process is rank `me` ----------------
  // s_n[g*E+e] = S[g,e,me]; receive rows: chunk_off[g] + prefix_e S[g,e',me]
  for (int i = tid; i < G * E; i += kLayThreads) {
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
  }
  __syncthreads();
  // send-side slot_base[me,e,d] = send_off[d] + sum_{e'<e} S[me,e',d]  (dest-major send buffer)
  if (w < G) {
    const int d = w;
    // send_off[d] = sum_{d'<d} sum_e S[me,e,d']
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
      if (e < E) slot_base[(me * E + e) * G + d] = running + incl - x;
      running += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  // per-expert work on me, residency, plan order
  for (int e = tid; e < E; e += kLayThreads) {
    int ne = 0, ns = 0;
    for (int g = 0; g < G; ++g) {
      const int v = s_n[g * E + e];
      ne += v;
      ns += (v > 0);
    }
    s_ne[e] = ne;
    s_nsrc[e] = ns;
  }
  __syncthreads();
  if (tid == 0) {
    s_scal[0] = 0;  // residents with work
    s_scal[1] = 0;  // home experts
    s_scal[2] = 0;  // experts with work
  }
  __syncthreads();
  for (int e = tid; e < E; e += kLayThreads) {
    const int ne = s_ne[e];
    const bool re = home[e] == me;
    if (re) atomicAdd(&s_scal[1], 1);
    if (ne > 0) {
      atomicAdd(&s_scal[2], 1);
      if (re) atomicAdd(&s_scal[0], 1);
      int pos = 0;
      for (int e2 = 0; e2 < E; ++e2) {
        const int n2 = s_ne[e2];
        if (n2 > 0 && plan_before(home[e2] == me, n2, e2, re, ne, e)) ++pos;
      }
      s_ord[e] = pos;
      s_cnt[pos] = s_nsrc[e];
    } else {
      s_ord[e] = -1;
    }
  }
  __syncthreads();
  const int n_work = s_scal[2];
  if (tid == 0) {
    int run = 0;
    for (int o = 0; o < n_work; ++o) {
      const int a = s_cnt[o];
      s_cnt[o] = run;
      run += a;
    }
    s_scal[3] = run;  // number of segments
    *n_seg_out = run;
    *n_fetch_out = n_work - s_scal[0];
  }
  __syncthreads();
  const int n_res_work = s_scal[0];
  const int n_home = s_scal[1];
  for (int e = tid; e < E; e += kLayThreads) {
    const int o = s_ord[e];
    if (o < 0) continue;
    int wslot;
    if (home[e] == me) {
      wslot = 0;
      for (int e2 = 0; e2 < e; ++e2) wslot += (home[e2] == me);
    } else {
      wslot = n_home + (o - n_res_work);
      fetch[o - n_res_work] = e;
    }
    int sidx = s_cnt[o];
    for (int g = 0; g < G; ++g) {
      const int v = s_n[g * E + e];
      if (v > 0) {
        segs[sidx] = make_int4(s_base[g] + s_off[g * E + e], v, wslot, e);
        ++sidx;
      }
    }
  }
  __syncthreads();
  // reuse s_off as per-segment m-tile counts
  const int n_seg = s_scal[3];
  for (int i = tid; i < n_seg; i += kLayThreads) s_off[i] = (segs[i].y + 127) / 128;
  __syncthreads();
  block_scan_to(s_off, n_seg, mprefix, s_tmp);
}

int launch_schedule(const int32_t* m_all, const int32_t* home, int G, int E, int q, int rebalance, int32_t* S,
                    int32_t* iters, int32_t* loads, cudaStream_t stream) {
  if (q < 1) return set_error(HM_EINVAL, "token threshold q must be >= 1");
  if (G < 1 || G > 32 || E < 1) return set_error(HM_EINVAL, "schedule: need 1 <= G <= 32 and E >= 1");
  const size_t sbytes = (size_t)G * E * G * sizeof(int);
  if (sbytes <= 200 * 1024) {
    cudaFuncSetAttribute(schedule_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes);
    schedule_kernel<true, false><<<1, 256, sbytes, stream>>>(m_all, home, G, E, q, rebalance, S, iters, loads);
  } else {
    schedule_kernel<false, false><<<1, 256, 0, stream>>>(m_all, home, G, E, q, rebalance, S, iters, loads);
  }
  return check_launch("schedule");
}

int launch_rebalance(int32_t* S, int G, int E, int q, int32_t* iters, int32_t* loads, cudaStream_t stream) {
  if (q < 1) return set_error(HM_EINVAL, "token threshold q must be >= 1");
  if (G < 1 || G > 32 || E < 1) return set_error(HM_EINVAL, "rebalance: need 1 <= G <= 32 and E >= 1");
  const size_t sbytes = (size_t)G * E * G * sizeof(int);
  if (sbytes <= 200 * 1024) {
    cudaFuncSetAttribute(schedule_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sbytes);
    schedule_kernel<true, true><<<1, 256, sbytes, stream>>>(nullptr, nullptr, G, E, q, 1, S, iters, loads);
  } else {
    schedule_kernel<false, true><<<1, 256, 0, stream>>>(nullptr, nullptr, G, E, q, 1, S, iters, loads);
  }
  return check_launch("rebalance");
}

int launch_layout(const int32_t* S, const int32_t* home, int G, int E, int mode, int me, int32_t* slot_base,
                  int32_t* segs, int32_t* n_seg, int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch,
                  cudaStream_t stream) {
  if (G < 1 || G > 32 || E < 1 || E > 1024 || G * E > kLayMaxGE)
    return set_error(HM_EINVAL, "dispatch_layout: need G <= 32, E <= 1024, G*E <= 8192");
  if (mode != HM_LAYOUT_LOCAL && mode != HM_LAYOUT_EP) return set_error(HM_EINVAL, "dispatch_layout: bad mode");
  if (mode == HM_LAYOUT_EP && (me < 0 || me >= G)) return set_error(HM_EINVAL, "dispatch_layout: bad rank");
  const size_t smem = (size_t)(3 * G * E + 1 + 3 * E) * sizeof(int);
  cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  layout_kernel<<<1, kLayThreads, smem, stream>>>(S, home, G, E, mode, me, slot_base, reinterpret_cast<int4*>(segs),
                                               n_seg, mtile_prefix, fetch, n_fetch);
  return check_launch("dispatch_layout");
}

}  // namespace hm
