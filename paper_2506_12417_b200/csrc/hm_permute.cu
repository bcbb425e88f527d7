// K4 (scatter/permute) and K7 (combine) - HBM-bound row movers.
//
// permute_kernel: Alg.1 step 4.  One warp per token: the
// token row is read ONCE into registers with 128-bit loads and written to each
// of its k scheduled rows with 128-bit stores.  The destination of the r-th
// assignment of (source g, expert e) is the first d with cumsum_d S[g,e,d] > r
// (split-bucket contract; the reference leaves token
// identity out).  r = tile_off + lrank comes from the router's
// deterministic rank pass, so the scatter is bit-reproducible.
//
// combine_kernel: Alg.1 step 6 + reconstruct.
// y[t] = sum_j w[t,j] * Y[pos[t,j]], fp32 multiply and add with explicit
// round-to-nearest (no FMA contraction) in slot order j = 0..k-1, bf16 output;
// the CPU oracle performs the identical float32 operation sequence.
#include "hm_common.cuh"
#include "hm_internal.h"

namespace hm {

constexpr int kPermWarps = 8;

template <int VEC>
__global__ void __launch_bounds__(kPermWarps * 32)
    permute_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ topk_idx,
                   const int32_t* __restrict__ lrank, const int32_t* __restrict__ tile_off,
                   const int32_t* __restrict__ S, const int32_t* __restrict__ slot_base, int64_t T,
                   int tokens_per_rank, int tiles_per_rank, int src_rank_base, int G, int E, int k, int n16,
                   uint4* __restrict__ out, int32_t* __restrict__ pos, int32_t* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kPermWarps + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lr = (int)(t / tokens_per_rank);
  const int tin = (int)(t - (int64_t)lr * tokens_per_rank);
  const int g = src_rank_base + lr;
  const int tile = lr * tiles_per_rank + tin / 128;

  uint4 v[VEC];
  const uint4* src = x + t * n16;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = i * 32 + lane;
    if (c < n16) v[i] = ld_global_nc_v4(src + c);
  }
  // lane j < k resolves slot j's buffer row (expert -> rank -> split-bucket destination ->
  // row): the k dependent load chains run side by side instead of one after another
  int pj = 0;
  if (lane < k) {
    const int j = lane;
    const int e = __ldg(topk_idx + t * k + j);
    const int r = __ldg(tile_off + (int64_t)tile * E + e) + __ldg(lrank + t * k + j);
    const int32_t* srow = S + ((int64_t)g * E + e) * G;
    int c = 0, d = 0;
    for (; d < G - 1; ++d) {
      const int s = __ldg(srow + d);
      if (c + s > r) break;
      c += s;
    }
    pj = __ldg(slot_base + ((int64_t)g * E + e) * G + d) + (r - c);
    pos[t * k + j] = pj;
    if (inv != nullptr) inv[pj] = (int32_t)(t * k + j);
  }
  for (int j = 0; j < k; ++j) {
    const int64_t p = __shfl_sync(0xffffffffu, pj, j);
    uint4* dst = out + p * n16;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int cc = i * 32 + lane;
      if (cc < n16) dst[cc] = v[i];
    }
  }
}

// Index-only scatter (the rows are gathered later by the FFN1 GEMM's TMA gather4):
// one thread per assignment computes its buffer row and the inverse map.
__global__ void __launch_bounds__(256)
    permute_index_kernel(const int32_t* __restrict__ topk_idx, const int32_t* __restrict__ lrank,
                         const int32_t* __restrict__ tile_off, const int32_t* __restrict__ S,
                         const int32_t* __restrict__ slot_base, int64_t n_assign, int k, int tokens_per_rank,
                         int tiles_per_rank, int src_rank_base, int G, int E, int32_t* __restrict__ pos,
                         int32_t* __restrict__ inv) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_assign) return;
  const int64_t t = a / k;
  const int lr = (int)(t / tokens_per_rank);
  const int tin = (int)(t - (int64_t)lr * tokens_per_rank);
  const int g = src_rank_base + lr;
  const int tile = lr * tiles_per_rank + tin / 128;
  const int e = __ldg(topk_idx + a);
  const int r = __ldg(tile_off + (int64_t)tile * E + e) + __ldg(lrank + a);
  const int32_t* srow = S + ((int64_t)g * E + e) * G;
  int c = 0, d = 0;
  for (; d < G - 1; ++d) {
    const int s = __ldg(srow + d);
    if (c + s > r) break;
    c += s;
  }
  const int p = __ldg(slot_base + ((int64_t)g * E + e) * G + d) + (r - c);
  pos[a] = p;
  if (inv != nullptr) inv[p] = (int32_t)a;
}

// Gather combine: rows addressed through pos (EP path: rows come back through the
// all_to_all in the send layout).
template <int VEC>
__global__ void __launch_bounds__(kPermWarps * 32)
    combine_kernel(const uint4* __restrict__ Y, const int32_t* __restrict__ pos, const float* __restrict__ w,
                   int64_t T, int k, int n16, const uint4* __restrict__ residual, uint4* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * kPermWarps + (threadIdx.x >> 5);
  if (t >= T) return;
  float acc[VEC][8];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = i * 32 + lane;
    if (residual != nullptr && c < n16) {
      const uint4 rv = ld_global_nc_v4(residual + t * n16 + c);
      const uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        acc[i][2 * h] = bf16lo(rr[h]);
        acc[i][2 * h + 1] = bf16hi(rr[h]);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 8; ++h) acc[i][h] = 0.0f;
    }
  }
  for (int j = 0; j < k; ++j) {
    const int64_t p = __ldg(pos + t * k + j);
    const float wj = __ldg(w + t * k + j);
    const uint4* row = Y + p * n16;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      const int c = i * 32 + lane;
      if (c < n16) {
        const uint4 u = ld_global_nc_v4(row + c);
        const uint32_t uu[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          acc[i][2 * h] = __fadd_rn(acc[i][2 * h], __fmul_rn(wj, bf16lo(uu[h])));
          acc[i][2 * h + 1] = __fadd_rn(acc[i][2 * h + 1], __fmul_rn(wj, bf16hi(uu[h])));
        }
      }
    }
  }
  uint4* dst = y + t * n16;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = i * 32 + lane;
    if (c < n16)
      dst[c] = make_uint4(pack_bf16x2(acc[i][0], acc[i][1]), pack_bf16x2(acc[i][2], acc[i][3]),
                          pack_bf16x2(acc[i][4], acc[i][5]), pack_bf16x2(acc[i][6], acc[i][7]));
  }
}

// Dense combine: Y is token-major [T*k, d] (the FFN2 epilogue scattered its rows there),
// so token t's k rows are one contiguous k*d*2-byte block.  One warp per token; for every
// 16-byte column chunk the k row loads are issued back to back (KT unrolled).
#ifndef HM_COMBINE_WARPS
#define HM_COMBINE_WARPS kPermWarps
#define HM_COMBINE_MINB 1
#else
#ifndef HM_COMBINE_MINB
#define HM_COMBINE_MINB (44 / HM_COMBINE_WARPS)  // <= 46 registers: a warp fits on an SMSP beside 3 GEMM warps
#endif
#define HM_COMBINE_CORUN 1
#endif
constexpr int kCombWarps = HM_COMBINE_WARPS;

template <int KT>
__global__ void __launch_bounds__(kCombWarps * 32, HM_COMBINE_MINB)
    combine_dense_kernel(const uint4* __restrict__ Y, const float* __restrict__ w, int64_t T, int k, int n16,
                         const uint4* __restrict__ residual, uint4* __restrict__ y, int parts) {
  // warp (t, part): token t's 16-byte column chunks [part*32, ...) step 32*parts.  parts > 1 for
  // small batches, so enough warps are in flight to cover DRAM latency
  const int lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * kCombWarps + (threadIdx.x >> 5);
  const int64_t t = wg / parts;
  const int part = (int)(wg - t * parts);
  if (t >= T) return;
  const int kk = KT > 0 ? KT : k;
  float wj[KT > 0 ? KT : 16];
#pragma unroll
  for (int j = 0; j < (KT > 0 ? KT : 16); ++j) wj[j] = (j < kk) ? __ldg(w + t * kk + j) : 0.0f;
  const uint4* base = Y + t * kk * n16;
  uint4* dst = y + t * n16;
  for (int c = part * 32 + lane; c < n16; c += 32 * parts) {
    uint4 u[KT > 0 ? KT : 16];
#pragma unroll
    for (int j = 0; j < (KT > 0 ? KT : 16); ++j)
      if (j < kk) u[j] = ld_global_nc_v4(base + (int64_t)j * n16 + c);
    float acc[8];
    if (residual != nullptr) {
      // decoder residual fused in: y = x + sum_j w_j Y_j (accumulation starts from x)
      const uint4 rv = ld_global_nc_v4(residual + t * n16 + c);
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
#pragma unroll
    for (int j = 0; j < (KT > 0 ? KT : 16); ++j) {
      if (j < kk) {
        const uint32_t uu[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          acc[2 * h] = __fadd_rn(acc[2 * h], __fmul_rn(wj[j], bf16lo(uu[h])));
          acc[2 * h + 1] = __fadd_rn(acc[2 * h + 1], __fmul_rn(wj[j], bf16hi(uu[h])));
        }
      }
    }
    dst[c] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                        pack_bf16x2(acc[6], acc[7]));
  }
}

int launch_permute(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
                   const int32_t* S, const int32_t* slot_base, int n_ranks, int tokens_per_rank, int src_rank_base,
                   int G, int E, int k, int d, void* out, int32_t* pos, int32_t* inv, cudaStream_t stream) {
  if (d <= 0 || d % 8 != 0 || d > 8192) return set_error(HM_EINVAL, "permute: need d %% 8 == 0 and d <= 8192");
  if (n_ranks < 1 || tokens_per_rank < 0 || G < 1 || E < 1 || k < 1 || k > 32)
    return set_error(HM_EINVAL, "permute: bad sizes (1 <= k <= 32)");
  const int64_t T = (int64_t)n_ranks * tokens_per_rank;
  if (T == 0) return HM_OK;
  const int n16 = d / 8;
  const int vec = (n16 + 31) / 32;
  const int tiles_per_rank = (tokens_per_rank + 127) / 128;
  if (out == nullptr) {
    const int64_t n_assign = T * k;
    permute_index_kernel<<<(unsigned)((n_assign + 255) / 256), 256, 0, stream>>>(
        topk_idx, lrank, tile_off, S, slot_base, n_assign, k, tokens_per_rank, tiles_per_rank, src_rank_base, G, E,
        pos, inv);
    return check_launch("permute_index");
  }
  const unsigned grid = (unsigned)((T + kPermWarps - 1) / kPermWarps);
  auto* xs = reinterpret_cast<const uint4*>(x);
  auto* o = reinterpret_cast<uint4*>(out);
#define HM_PERM(V)                                                                                              \
  permute_kernel<V><<<grid, kPermWarps * 32, 0, stream>>>(xs, topk_idx, lrank, tile_off, S, slot_base, T,       \
                                                          tokens_per_rank, tiles_per_rank, src_rank_base, G, E, \
                                                          k, n16, o, pos, inv)
  if (vec <= 1) HM_PERM(1);
  else if (vec <= 2) HM_PERM(2);
  else if (vec <= 4) HM_PERM(4);
  else if (vec <= 8) HM_PERM(8);
  else if (vec <= 16) HM_PERM(16);
  else HM_PERM(32);
#undef HM_PERM
  return check_launch("permute");
}

int launch_combine(const void* Y, const int32_t* pos, const float* topk_w, int T, int k, int d, const void* residual,
                   void* y, cudaStream_t stream) {
  if (d <= 0 || d % 8 != 0 || d > 8192) return set_error(HM_EINVAL, "combine: need d %% 8 == 0 and d <= 8192");
  if (T < 0 || k < 1) return set_error(HM_EINVAL, "combine: bad sizes");
  if (T == 0) return HM_OK;
  const int n16 = d / 8;
  const int vec = (n16 + 31) / 32;
  const unsigned grid = (unsigned)((T + kPermWarps - 1) / kPermWarps);
  // dense layout: split each token's columns over up to n16/32 warps until ~16K warps are in flight
  int parts = 1;
  while (parts * 2 <= (n16 + 31) / 32 && (int64_t)T * parts * 2 <= 16384) parts *= 2;
  const unsigned grid_d = (unsigned)(((int64_t)T * parts + kCombWarps - 1) / kCombWarps);
  auto* Ys = reinterpret_cast<const uint4*>(Y);
  auto* o = reinterpret_cast<uint4*>(y);
  auto* res = reinterpret_cast<const uint4*>(residual);
  if (pos == nullptr) {
    if (k > 16) return set_error(HM_EINVAL, "combine: dense layout needs k <= 16");
#ifdef HM_COMBINE_CORUN
#define HM_DENSE_ATTR(KT) \
  cudaFuncSetAttribute(combine_dense_kernel<KT>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#else
#define HM_DENSE_ATTR(KT)
#endif
#define HM_DENSE(KT)                                                                                  \
  do {                                                                                                \
    HM_DENSE_ATTR(KT)                                                                                 \
    combine_dense_kernel<KT><<<grid_d, kCombWarps * 32, 0, stream>>>(Ys, topk_w, T, k, n16, res, o, parts); \
  } while (0)
    if (k == 1) HM_DENSE(1);
    else if (k == 2) HM_DENSE(2);
    else if (k == 4) HM_DENSE(4);
    else if (k == 8) HM_DENSE(8);
    else HM_DENSE(0);
#undef HM_DENSE
    return check_launch("combine_dense");
  }
#define HM_COMB(V) combine_kernel<V><<<grid, kPermWarps * 32, 0, stream>>>(Ys, pos, topk_w, T, k, n16, res, o)
  if (vec <= 1) HM_COMB(1);
  else if (vec <= 2) HM_COMB(2);
  else if (vec <= 4) HM_COMB(4);
  else if (vec <= 8) HM_COMB(8);
  else if (vec <= 16) HM_COMB(16);
  else HM_COMB(32);
#undef HM_COMB
  return check_launch("combine");
}

}  // namespace hm
