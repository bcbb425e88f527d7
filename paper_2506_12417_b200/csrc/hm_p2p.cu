// Expert parallelism over NVSwitch peer memory: one-sided, no host synchronisation.
//
// The NCCL path (ep.py, transport "nccl") needs S on the host for the all_to_all split
// sizes.  With every rank's buffers mapped into every other rank (CUDA IPC, once at set-up)
// the replicated schedule S is all a sender needs to place its rows directly in the
// receiver's buffer ("a one-sided push using the replicated S needs no
// host-side count exchange"):
//
//   ep_offsets_kernel    flows = S.sum(e); per destination d the delta between this rank's
//                        send-layout row and the row of the same assignment in d's receive
//                        buffer ([source][expert][rank], hm_sched.cu dev_layout EP mode), and
//                        the receive-row split per source.
//   dispatch_push_kernel K4 fused with the dispatch all-to-all: each token row is read once
//                        and stored (128-bit, NVLink) into every scheduled destination's
//                        receive buffer, with its token-major index (t*k + j) beside it.
//   fetch_kernel         K6 driven from the device: copies the plan's fetch list (peer HBM
//                        over NVLink, or pinned host memory) into the cache slots in plan
//                        order and publishes a ready flag per expert (the FFN GEMM producer
//                        waits per expert), so the fetch list never visits the host.  (A
//                        bounded cache is fetched by pairs inside the GEMM launch instead,
//                        hm_gemm.cu, so fetch and GEMM are co-resident by construction.)
//
// The FFN2 GEMM stores its rows straight into the source rank's token-major output
// (hm_gemm.cu remote epilogue), which is the combine all-to-all fused into the GEMM.
#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

// ------------------------------------------------------------------------------------------
// offsets: dst_delta[d] = (sum_{g<me} flows[g][d]) - (sum_{d'<d} flows[me][d'])
//          recv_split[g] = sum_{g'<g} flows[g'][me]   (g = 0..G)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
    ep_offsets_kernel(const int32_t* __restrict__ S, int G, int E, int me, int32_t* __restrict__ dst_delta,
                      int32_t* __restrict__ recv_split) {
  __shared__ int flows[32 * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // one warp per (g, d) pair: flows[g][d] = sum_e S[g,e,d]
  for (int p = w; p < G * G; p += nw) {
    const int g = p / G, d = p - (p / G) * G;
    int s = 0;
    for (int e = lane; e < E; e += 32) s += __ldg(S + ((int64_t)g * E + e) * G + d);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) flows[p] = s;
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int d = threadIdx.x;
    int recv_off = 0, send_off = 0;
    for (int g = 0; g < me; ++g) recv_off += flows[g * G + d];
    for (int d2 = 0; d2 < d; ++d2) send_off += flows[me * G + d2];
    dst_delta[d] = recv_off - send_off;
  }
  if (threadIdx.x == 0) {
    int run = 0;
    for (int g = 0; g < G; ++g) {
      recv_split[g] = run;
      run += flows[g * G + me];
    }
    recv_split[G] = run;
  }
}

// ------------------------------------------------------------------------------------------
// dispatch push: permute_kernel's row placement (hm_permute.cu) with the store going to the
// destination rank's receive buffer instead of a local send buffer
// ------------------------------------------------------------------------------------------
constexpr int kPushWarps = 8;

template <int VEC>
__global__ void __launch_bounds__(kPushWarps * 32)
    dispatch_push_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ topk_idx,
                         const int32_t* __restrict__ lrank, const int32_t* __restrict__ tile_off,
                         const int32_t* __restrict__ S, const int32_t* __restrict__ slot_base,
                         const int32_t* __restrict__ dst_delta, int64_t T, int me, int G, int E, int k, int n16,
                         const unsigned long long* __restrict__ dst_rows, const unsigned long long* __restrict__ dst_tok,
                         int32_t* __restrict__ pos) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kPushWarps + (threadIdx.x >> 5);
  if (t >= T) return;
  const int tile = (int)(t / 128);
  uint4 v[VEC];
  const uint4* src = x + t * n16;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = i * 32 + lane;
    if (c < n16) v[i] = ld_global_nc_v4(src + c);
  }
  // lane j < k resolves slot j's destination rank and receive row (the k dependent load
  // chains side by side); the row stores below then only need two shuffles per slot
  int qj = 0, dj = 0;
  if (lane < k) {
    const int j = lane;
    const int e = __ldg(topk_idx + t * k + j);
    const int r = __ldg(tile_off + (int64_t)tile * E + e) + __ldg(lrank + t * k + j);
    const int32_t* srow = S + ((int64_t)me * E + e) * G;
    int c = 0, d = 0;
    for (; d < G - 1; ++d) {
      const int s = __ldg(srow + d);
      if (c + s > r) break;
      c += s;
    }
    const int p = __ldg(slot_base + ((int64_t)me * E + e) * G + d) + (r - c);
    if (dst_delta != nullptr) {  // HM_LAYOUT_EP: p is the send-layout row, shifted into d's buffer
      qj = p + __ldg(dst_delta + d);
      reinterpret_cast<int32_t*>(__ldg(dst_tok + d))[qj] = (int32_t)(t * k + j);
    } else {  // HM_LAYOUT_EP_EXPERT: p is already the row in d's buffer; tag the row with its source
      qj = p;
      reinterpret_cast<int32_t*>(__ldg(dst_tok + d))[qj] = (int32_t)(((uint32_t)me << 24) | (uint32_t)(t * k + j));
    }
    dj = d;
    if (pos != nullptr) pos[t * k + j] = p;
  }
  for (int j = 0; j < k; ++j) {
    const int64_t q = __shfl_sync(0xffffffffu, qj, j);
    const int d = __shfl_sync(0xffffffffu, dj, j);
    uint4* dst = reinterpret_cast<uint4*>(__ldg(dst_rows + d)) + q * n16;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int cc = i * 32 + lane;
      if (cc < n16) dst[cc] = v[i];
    }
  }
}

// ------------------------------------------------------------------------------------------
// expert-ordered dispatch push (overlapped with FFN1).  The unordered push above finishes every
// expert's rows at about the same time (token order), so FFN1 can only start after the whole
// all-to-all.  Here every sender walks its work list in the DESTINATIONS' plan order (item
// p*G + d = its bucket of the p-th expert of destination d, hm_plan_dispatch), 8 rows per work
// unit, and after each unit adds the row count to the destination's per-expert arrival counter
// (system-scope release after the rows).  FFN1 is launched right behind this kernel with
// programmatic dependent launch and its producer waits per segment for arrive[e] == rows of e,
// so the first experts' tiles start while later experts are still in flight over NVLink.
//   phase 1: order[ebase[e] + r] = t*k + j for this rank's r-th assignment to e (and pos);
//   grid barrier (all CTAs resident: launched on dedicated TPCs before its dependent GEMM);
//   phase 2: 8-row units (one warp each) dealt round-robin in (position, destination) order.
// ------------------------------------------------------------------------------------------
// One CTA per SM of 4 warps (one per SM sub-partition) of <= 64 registers, so that the FFN1 pair
// CTA launched behind it with PDL fits beside it: each sub-partition has 16K registers and the
// GEMM CTA holds 3 warps x 4,608 of them on two of its sub-partitions; the push also asks for the
// maximal shared-memory carveout (tools/pdl_probe: the GEMM's CTAs then start ~3 us after the
// push instead of after it).  Measured alternative: the push on 4-16 dedicated TPCs of full-SM
// CTAs (GEMM on the others) - 93-241 us for one rank's rows, far slower.
constexpr int kOPushThreads = 128;
// rows per work unit (one warp, one arrival increment).  Units are dealt round-robin over the
// grid's warps, so ~#warps units are in flight at once: small units keep the completion order
// close to the plan order (the first experts land after ~1/4 of the push, not at its end)
constexpr int kOPushRows = 8;

template <int VEC>
__global__ void __launch_bounds__(kOPushThreads, 8)  // <= 64 registers: co-resident with the FFN1 pairs
    dispatch_push_ordered_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ topk_idx,
                                 const int32_t* __restrict__ lrank, const int32_t* __restrict__ tile_off,
                                 const int32_t* __restrict__ S, const int32_t* __restrict__ slot_base,
                                 const int4* __restrict__ items, const int32_t* __restrict__ cprefix,
                                 const int32_t* __restrict__ ebase, int n_items, int64_t T, int me, int G, int E,
                                 int k, int n16, const unsigned long long* __restrict__ dst_rows,
                                 const unsigned long long* __restrict__ dst_tok,
                                 const unsigned long long* __restrict__ dst_arrive, int32_t* __restrict__ order,
                                 int32_t* __restrict__ pos, unsigned* __restrict__ sync) {
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // ---- phase 1: per-expert assignment order (+ pos: the row of each assignment in its
  // destination's receive buffer, as the unordered push reports it)
  const int64_t TK = T * k;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < TK; a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = a / k;
    const int e = __ldg(topk_idx + a);
    const int r = __ldg(tile_off + (t / 128) * E + e) + __ldg(lrank + a);
    order[__ldg(ebase + e) + r] = (int32_t)a;
    if (pos != nullptr) {
      const int32_t* srow = S + ((int64_t)me * E + e) * G;
      int c = 0, d = 0;
      for (; d < G - 1; ++d) {
        const int sv = __ldg(srow + d);
        if (c + sv > r) break;
        c += sv;
      }
      pos[a] = __ldg(slot_base + ((int64_t)me * E + e) * G + d) + (r - c);
    }
  }
  // ---- grid barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(sync, 1u);
    long long spins = 0;
    while (ld_acquire_gpu(reinterpret_cast<const int*>(sync)) < (int)gridDim.x) {
      __nanosleep(32);
      if (++spins > (1ll << 26)) {
        printf("hm dispatch_push_ordered: grid barrier timed out (CTAs not co-resident)\n");
        __trap();
      }
    }
  }
  __syncthreads();
#ifdef HM_OPUSH_ONLY_P1  // diagnostics: phase 1 + barrier only
  return;
#endif
  const int total = __ldcg(cprefix + n_items);
  if (total < 0) {
    if (threadIdx.x == 0) printf("hm dispatch_push_ordered: no push work list (planner took the general path)\n");
    __trap();
  }
  // ---- phase 2: 8-row units in (position, destination) order, one warp per unit (the release
  // after a unit stalls only its warp), dealt round-robin over the grid's warps in order
  const int nwarps = gridDim.x * (kOPushThreads / 32);
  int it = 0;  // item of the warp's current unit: units only grow, so the search moves forward
  for (int u = blockIdx.x * (kOPushThreads / 32) + warp; u < total; u += nwarps) {
    // 32-ary search from the previous item (cprefix is non-decreasing, so the lanes whose probe
    // is <= u are a prefix): each step narrows the range 32-fold with one coalesced probe
    for (int span = n_items - it; span > 0;) {
      const int step = (span + 31) >> 5;
      const int j = it + (lane + 1) * step;
      const unsigned b = __ballot_sync(0xffffffffu, j <= n_items && __ldg(cprefix + j) <= u);
      const int n = __popc(b);
      it += n * step;
      span = (n == 32 ? span - 32 * step : step - 1);
      if (step == 1) break;
    }
    const int4 item = __ldg(items + it);
    const int d = it & (G - 1);
    const int r0 = (u - __ldg(cprefix + it)) * kOPushRows;
    const int nr = min(kOPushRows, item.z - r0);
    const int e = item.x;
    const int ob = __ldg(ebase + e) + item.y + r0;
    uint4* dst = reinterpret_cast<uint4*>(__ldg(dst_rows + d)) + (int64_t)(item.w + r0) * n16;
    int32_t* tok = reinterpret_cast<int32_t*>(__ldg(dst_tok + d));
    const int my_a = lane < nr ? __ldcg(order + ob + lane) : 0;  // the unit's assignment indices
#ifdef HM_OPUSH_NO_ROWS  // diagnostics: work distribution + counts only
#ifdef HM_OPUSH_GPU_SCOPE
    if (lane == 0) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(reinterpret_cast<int*>(__ldg(dst_arrive + d)) + e), "r"(nr) : "memory");
#else
    if (lane == 0) red_release_sys_add(reinterpret_cast<int*>(__ldg(dst_arrive + d)) + e, nr);
#endif
    continue;
#endif
    for (int rr = 0; rr < nr; ++rr) {  // a row's VEC 16-byte loads per lane in flight, then its stores
      const int a = __shfl_sync(0xffffffffu, my_a, rr);
      const uint4* src = x + (int64_t)(a / k) * n16;
      uint4 v[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const int c = i * 32 + lane;
        if (c < n16) v[i] = ld_global_nc_v4(src + c);
      }
      uint4* drow = dst + (int64_t)rr * n16;
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const int c = i * 32 + lane;
        if (c < n16) drow[c] = v[i];
      }
    }
    if (lane < nr) tok[item.w + r0 + lane] = (int32_t)(((uint32_t)me << 24) | (uint32_t)my_a);
    // every lane's rows (ordered before lane 0 by the warp barrier) before the count: the
    // release is cumulative over them
    __syncwarp();
    if (lane == 0) {
      int* cnt = reinterpret_cast<int*>(__ldg(dst_arrive + d)) + e;
#ifdef HM_OPUSH_GPU_SCOPE
      if (true)
#else
      if (d == me)  // this GPU's own buffer: device scope suffices (its FFN1 reads it)
#endif
        asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(cnt), "r"(nr) : "memory");
      else
        red_release_sys_add(cnt, nr);
    }
  }
}

// ------------------------------------------------------------------------------------------
// device-driven expert fetch (K6).  All CTAs copy fetch i's gate/up block, then its down
// block, then move on (one logical channel in plan order, engine.py:253-265); the last CTA
// to finish a block publishes its slot's ready flag with release semantics.
// ------------------------------------------------------------------------------------------
// One 4-warp CTA per SM, <= 64 registers, maximal shared-memory carveout: the fetch runs beside
// FFN1 (its own stream) on every SM instead of taking SMs from the persistent GEMM's pairs (a
// 512-thread CTA does not fit beside a GEMM pair CTA: 16K registers per SM sub-partition, 3 GEMM
// warps x 4,608 on two of them; its SMs' pairs then waited for the whole fetch).  8 x 16 B per
// lane in flight: ~2.4 MB per GPU, enough for NVLink's latency-bandwidth product.
#ifndef HM_FETCH_UNROLL
#define HM_FETCH_UNROLL 8
#endif
#ifdef HM_FETCH_WIDE  // A/B: the round-1 configuration (32 CTAs x 512 threads, 4 x 16 B in flight)
constexpr int kFetchThreads = 512;
constexpr int kFetchUnroll = 4;
#else
constexpr int kFetchThreads = 128;
constexpr int kFetchUnroll = HM_FETCH_UNROLL;
#endif

__device__ __forceinline__ void copy_block(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kFetchUnroll - 1) * stride < n16; i += kFetchUnroll * stride) {
    uint4 v[kFetchUnroll];
#pragma unroll
    for (int u = 0; u < kFetchUnroll; ++u) v[u] = ld_global_nc_v4(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < kFetchUnroll; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = ld_global_nc_v4(src + i);
}

__device__ __forceinline__ void block_done(int32_t* counter, int32_t* flag, int value) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int old = atomicAdd(counter, 1);
    if (old == (int)gridDim.x - 1) {
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
    }
  }
}

__global__ void __launch_bounds__(kFetchThreads, 2048 / kFetchThreads)
    fetch_kernel(const int32_t* __restrict__ fetch, const int32_t* __restrict__ n_fetch_p,
                 const unsigned long long* __restrict__ src_in, const unsigned long long* __restrict__ src_out,
                 int64_t in16, int64_t out16, uint4* __restrict__ dst_in, uint4* __restrict__ dst_out, int first_slot,
                 int n_slots, int32_t* __restrict__ ready_in, int32_t* __restrict__ ready_out,
                 int32_t* __restrict__ counters, int n_counters, int value) {
  const int n_fetch = *n_fetch_p;
  // more fetches than slots (a bounded cache belongs to the in-GEMM fetch pairs, hm_gemm.cu):
  // fail the launch loudly rather than leave the GEMM waiting on (or reading) unfilled slots
  if (n_fetch > n_slots || 2 * n_fetch > n_counters) __trap();
  // every gate/up block first (all FFN1 waits on), then the down blocks (FFN2's), each in plan order
  for (int i = 0; i < n_fetch; ++i) {
    const int e = __ldg(fetch + i);
    copy_block(dst_in + (int64_t)(first_slot + i) * in16, reinterpret_cast<const uint4*>(__ldg(src_in + e)), in16);
    block_done(counters + 2 * i, ready_in + e, value);
  }
  for (int i = 0; i < n_fetch; ++i) {
    const int e = __ldg(fetch + i);
    copy_block(dst_out + (int64_t)(first_slot + i) * out16, reinterpret_cast<const uint4*>(__ldg(src_out + e)),
               out16);
    block_done(counters + 2 * i + 1, ready_out + e, value);
  }
}

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------
int launch_ep_offsets(const int32_t* S, int G, int E, int me, int32_t* dst_delta, int32_t* recv_split,
                      cudaStream_t stream) {
  if (G < 1 || G > 32 || E < 1 || me < 0 || me >= G) return set_error(HM_EINVAL, "ep_offsets: bad G/E/me");
  ep_offsets_kernel<<<1, 1024, 0, stream>>>(S, G, E, me, dst_delta, recv_split);
  return check_launch("ep_offsets");
}

int launch_dispatch_push(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
                         const int32_t* S, const int32_t* slot_base, const int32_t* dst_delta, int tokens, int me,
                         int G, int E, int k, int d, const unsigned long long* dst_rows,
                         const unsigned long long* dst_tok, int32_t* pos, cudaStream_t stream) {
  if (d % 8 != 0) return set_error(HM_EINVAL, "dispatch_push: d must be a multiple of 8");
  if (G < 1 || G > 32 || me < 0 || me >= G || k < 1 || k > 32)
    return set_error(HM_EINVAL, "dispatch_push: bad G/me/k");
  if (dst_delta == nullptr && (int64_t)tokens * k > (1 << 24))
    return set_error(HM_EINVAL, "dispatch_push: tagged rows need tokens * k <= 2^24");
  if (tokens <= 0) return HM_OK;
  const int n16 = d / 8;
  const int blocks = (tokens + kPushWarps - 1) / kPushWarps;
  const auto* xs = reinterpret_cast<const uint4*>(x);
#define HM_PUSH(V)                                                                                             \
  dispatch_push_kernel<V><<<blocks, kPushWarps * 32, 0, stream>>>(xs, topk_idx, lrank, tile_off, S, slot_base, \
                                                                  dst_delta, tokens, me, G, E, k, n16,          \
                                                                  dst_rows, dst_tok, pos)
  if (n16 <= 32) HM_PUSH(1);
  else if (n16 <= 64) HM_PUSH(2);
  else if (n16 <= 128) HM_PUSH(4);
  else if (n16 <= 256) HM_PUSH(8);
  else if (n16 <= 512) HM_PUSH(16);
  else return set_error(HM_EINVAL, "dispatch_push: d > 4096 unsupported");
#undef HM_PUSH
  return check_launch("dispatch_push");
}

int launch_dispatch_push_ordered(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
                                 const int32_t* S, const int32_t* slot_base, const int32_t* items,
                                 const int32_t* cprefix, const int32_t* ebase, int tokens, int me, int G, int E, int k,
                                 int d, const unsigned long long* dst_rows, const unsigned long long* dst_tok,
                                 const unsigned long long* dst_arrive, int32_t* order, int32_t* pos, uint32_t* sync,
                                 cudaStream_t stream) {
  if (d % 8 != 0) return set_error(HM_EINVAL, "dispatch_push_ordered: d must be a multiple of 8");
  if (G < 1 || G > 32 || (G & (G - 1)) != 0 || me < 0 || me >= G || k < 1 || k > 32)
    return set_error(HM_EINVAL, "dispatch_push_ordered: bad G (power of two <= 32) / me / k");
  if ((int64_t)tokens * k > (1 << 24))
    return set_error(HM_EINVAL, "dispatch_push_ordered: tagged rows need tokens * k <= 2^24");
  if (items == nullptr || cprefix == nullptr || ebase == nullptr || dst_arrive == nullptr || order == nullptr ||
      sync == nullptr)
    return set_error(HM_EINVAL, "dispatch_push_ordered: work list, arrival counters, order and sync are required");
  // the grid barrier needs every CTA resident: one per SM (the kernel runs before its dependent GEMM)
  cudaError_t ce = cudaMemsetAsync(sync, 0, 2 * sizeof(uint32_t), stream);
  if (ce != cudaSuccess) return set_error(HM_ECUDA, "dispatch_push_ordered sync: %s", cudaGetErrorString(ce));
  if (tokens < 0) return set_error(HM_EINVAL, "dispatch_push_ordered: tokens must be >= 0");
  const int n16 = d / 8;
  const int grid = num_sms();
  const auto* xs = reinterpret_cast<const uint4*>(x);
  const int4* it4 = reinterpret_cast<const int4*>(items);
  // maximal shared-memory carveout: an SM configured for this kernel's (tiny) shared memory could
  // not take the FFN1 CTAs (~224 KB) launched behind it until the push left the SM
  cudaError_t le = cudaSuccess;
#define HM_OPUSH(V)                                                                                              \
  do {                                                                                                           \
    cudaFuncSetAttribute(dispatch_push_ordered_kernel<V>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  \
    dispatch_push_ordered_kernel<V><<<grid, kOPushThreads, 0, stream>>>(                                         \
        xs, topk_idx, lrank, tile_off, S, slot_base, it4, cprefix, ebase, G * E, tokens, me, G, E, k, n16,        \
        dst_rows, dst_tok, dst_arrive, order, pos, reinterpret_cast<unsigned*>(sync));                           \
    le = cudaGetLastError();                                                                                     \
  } while (0)
  if (n16 <= 32) HM_OPUSH(1);
  else if (n16 <= 64) HM_OPUSH(2);
  else if (n16 <= 128) HM_OPUSH(4);
  else if (n16 <= 256) HM_OPUSH(8);
  else if (n16 <= 512) HM_OPUSH(16);
  else return set_error(HM_EINVAL, "dispatch_push_ordered: d > 4096 unsupported");
#undef HM_OPUSH
  if (le != cudaSuccess) return set_error(HM_ECUDA, "dispatch_push_ordered launch: %s", cudaGetErrorString(le));
  return check_launch("dispatch_push_ordered");
}

int launch_fetch_experts(const int32_t* fetch, const int32_t* n_fetch, const unsigned long long* src_in,
                         const unsigned long long* src_out, size_t in_bytes, size_t out_bytes, void* dst_in,
                         void* dst_out, int first_slot, int n_slots, int32_t* ready_in, int32_t* ready_out,
                         int32_t* counters, int n_counters, int value, int ctas, cudaStream_t stream) {
  if (in_bytes % 16 != 0 || out_bytes % 16 != 0) return set_error(HM_EINVAL, "fetch_experts: sizes must be 16-byte multiples");
  if (n_slots <= 0) return HM_OK;
  if (n_counters < 2) return set_error(HM_EINVAL, "fetch_experts: counters too small");
  cudaError_t e = cudaMemsetAsync(counters, 0, sizeof(int32_t) * n_counters, stream);
  if (e != cudaSuccess) return set_error(HM_ECUDA, "fetch_experts memset: %s", cudaGetErrorString(e));
#ifdef HM_FETCH_WIDE
  const int grid = ctas > 0 ? ctas : 32;
#else
  cudaFuncSetAttribute(fetch_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int grid = ctas > 0 ? ctas : num_sms();
#endif
  fetch_kernel<<<grid, kFetchThreads, 0, stream>>>(
      fetch, n_fetch, src_in, src_out, (int64_t)(in_bytes / 16), (int64_t)(out_bytes / 16),
      reinterpret_cast<uint4*>(dst_in), reinterpret_cast<uint4*>(dst_out), first_slot, n_slots, ready_in, ready_out,
      counters, n_counters, value);
  return check_launch("fetch_experts");
}

}  // namespace hm
