/*
 * harmoe.h - C ABI of the B200-native HarMoEny expert-parallel MoE block.
 *
 * libharmoe.so (paper_2506_12417_b200/libharmoe.so) exports exactly these
 * entry points.  Plain pointers and sizes only: every pointer argument is a
 * device pointer unless stated otherwise; `stream` is a cudaStream_t passed as
 * void*.  Every call is stream-ordered, never allocates, never synchronises the
 * host, and returns HM_OK (0) or an error code; hm_last_error() gives the
 * message.  There is no CPU fallback.
 *
 * Each entry point replaces one phase of the reference's MoE-layer path
 * (reference = /root/reference, moesim + PAPER.md Alg. 1):
 *
 *   hm_router_topk      Alg.1 step 1 "router"; the reference
 *                       stand-in is workload.sample_routing (workload.py:167-180)
 *   hm_hist_scan        per-GPU token->expert histogram = RoutingMatrix row
 *                       (core.py:89-96) = metadata m_expert
 *   hm_schedule /       initial_assign + rebalance (policies.py:109-171) as
 *   hm_rebalance        dispatched by engine.build_schedule (engine.py:287-299);
 *                       even_split_assign (policies.py:174-203) by policy code
 *   hm_schedule_batched build_schedule over every (batch, layer) of a trace
 *                       (engine.py:430-447; trace format workload.py:213-232)
 *   hm_dispatch_layout  byte flows of the scatter (engine._exchange_byte_vectors,
 *                       engine.py:278-284) + per-GPU execution order of
 *                       plan_gpu_execution (engine.py:233-234)
 *   hm_plan             steps 2-3 fused: histogram reduce + hm_schedule + layout
 *   hm_permute          Alg.1 step 4 scatter
 *   hm_grouped_gemm     Alg.1 step 5 expert compute (cost
 *                       model engine.py:128-132)
 *   hm_fetch_expert(s)  async expert fetch (engine.py:253-265)
 *   hm_combine          Alg.1 step 6 gather + reconstruct
 *   hm_grouped_gemm_combine  steps 5 (FFN2) + 6 fused: the combine runs in the FFN2 epilogue
 *   hm_ep_offsets, hm_dispatch_push, hm_grouped_gemm_remote, hm_stream_signal/wait,
 *   hm_ipc_*            expert parallelism over NVSwitch peer memory: the metadata exchange
 *                       and the scatter / gather all-to-alls of engine.py:328-375
 */
#ifndef HARMOE_H_
#define HARMOE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HM_API __attribute__((visibility("default")))
#else
#define HM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define HM_OK 0
#define HM_EINVAL 1  /* invalid argument (the Python layer raises ValueError) */
#define HM_ECUDA 2   /* CUDA runtime / driver error */
#define HM_ENCCL 3   /* reserved: collective error (collectives run in torch.distributed) */
#define HM_ENOSPC 4  /* a buffer capacity is too small */

/* grouped-GEMM epilogues */
#define HM_EPI_STORE 0  /* out = bf16(acc) */
#define HM_EPI_RELU 1   /* out = bf16(relu(acc)) (Switch FFN1) */
#define HM_EPI_SWIGLU 2 /* out = bf16(silu(gate) * up), W13 block-interleaved by 128 rows */

/* dispatch layouts */
/* scheduling policy (the `rebalance` argument of hm_schedule / hm_schedule_batched / hm_plan) */
#define HM_POLICY_NONE 0       /* initial_assign only (policies.py:109-117; SimFlags rebalancing off) */
#define HM_POLICY_REBALANCE 1  /* initial_assign + Alg. 2 rebalance (policies.py:120-141) */
#define HM_POLICY_EVEN_SPLIT 2 /* even_split_assign baseline (policies.py:174-203); ignores home and q */

#define HM_LAYOUT_LOCAL 0 /* all G ranks on this device: buffer [dest][expert][source][rank] */
#define HM_LAYOUT_EP 1    /* this process is rank `me`: send buffer [dest][expert][rank], */
                          /* receive buffer [source][expert][rank] (NCCL all_to_all chunks) */
#define HM_LAYOUT_EP_EXPERT 2 /* rank `me`, one-sided p2p dispatch: every rank's receive buffer is */
                              /* [expert][source][rank], slot_base[g,e,d] = that bucket's row in  */
                              /* rank d's buffer; one GEMM segment per expert (all sources)       */

/* diagnostics: %globaltimer stamps (ns) of the last hm_plan launch: start, after the histogram
 * reduce, after the schedule, after the layout (host buffer of 4 int64; synchronises the device).
 * Recorded only by a library built with -DHM_PLAN_PHASES (zeros otherwise). */
HM_API int hm_debug_plan_phases(long long* out4);

HM_API int hm_version(void);
HM_API const char* hm_last_error(void);
HM_API int hm_num_sms(void);
HM_API int hm_gemm_tile_m(void); /* rows per GEMM tile (128) */
/* CTA pairs of the 2-CTA grouped GEMM that fit on the device at once (its persistent grid) */
HM_API int hm_gemm_resident_pairs(int epilogue, int gather);

/*
 * Router (K1) + histogram/rank pass (K2), fused: one CTA per 128-token tile.
 *   x        [n_ranks*tokens_per_rank, d] bf16      token activations
 *   wg       [E_pad, d] bf16                         gate weights (nn.Linear layout),
 *                                                    E_pad = E rounded up to 16 (rows >= E are ignored)
 *   bias     [E] fp32 or NULL                        additive logit bias
 *   topk_idx [T, k] int32, topk_w [T, k] fp32       top-k over fp32 logits, lowest index wins ties;
 *                                                    weights = softmax probs (renormalised over k if set)
 *   tile_hist[n_ranks*tiles_per_rank, E] int32       per-tile expert histogram
 *   lrank    [T, k] int32                            rank of each assignment among same-expert
 *                                                    assignments of its tile, (token, slot) order
 * tiles_per_rank = ceil(tokens_per_rank / 128).  Requires d % 64 == 0, 1 <= k <= 16, k <= E <= 256.
 */
HM_API int hm_router_topk(const void* x, const void* wg, const float* bias, int n_ranks, int tokens_per_rank, int d,
                   int E, int k, int renormalize, int32_t* topk_idx, float* topk_w, int32_t* tile_hist,
                   int32_t* lrank, void* stream);

/* Per-rank histogram m_expert[n_ranks, E] and per-tile exclusive offsets tile_off (same shape as
 * tile_hist).  Row r of `hist` is RoutingMatrix.counts[r] (core.py:93-95). */
HM_API int hm_hist_scan(const int32_t* tile_hist, int n_ranks, int tiles_per_rank, int E, int32_t* hist,
                 int32_t* tile_off, void* stream);

/*
 * Scheduler (K3): S[g,e,home[e]] = m_all[g,e] (policies.py:109-117), then, when `rebalance`,
 * HarMoEny's greedy token rebalancing (policies.py:120-141, Alg. 2) with threshold q, bit-exact
 * against the reference (lowest-index ties).  Replicated on every rank; no communication.
 * `rebalance` is an HM_POLICY_* code (0/1 keep their boolean meaning); HM_POLICY_EVEN_SPLIT
 * builds the even_split_assign baseline schedule (policies.py:174-203) instead, iters = 0.
 *   m_all [G,E] int32, home [E] int32 -> S [G,E,G] int32, iters [1] int32, loads [G] int32 (or NULL).
 * q < 1 -> HM_EINVAL ("token threshold q must be >= 1").  Requires G <= 32.
 */
HM_API int hm_schedule(const int32_t* m_all, const int32_t* home, int G, int E, int q, int rebalance, int32_t* S,
                int32_t* iters, int32_t* loads, void* stream);

/*
 * Batched scheduler: B independent routing matrices m_all [B,G,E] (e.g. every layer of every
 * batch of a recorded trace, moesim trace format workload.py:213-232) scheduled by one launch,
 * one CTA per instance.  S [B,G,E,G], iters [B], loads [B,G] (or NULL).
 */
HM_API int hm_schedule_batched(const int32_t* m_all, const int32_t* home, int B, int G, int E, int q, int rebalance,
                               int32_t* S, int32_t* iters, int32_t* loads, void* stream);

/*
 * In-place rebalance of an arbitrary schedule S [G,E,G] int32 (policies.py:144-171, the
 * drop-in for moesim.rebalance / rebalance_with_stats).  Same tie and stop rules as hm_schedule.
 */
HM_API int hm_rebalance(int32_t* S, int G, int E, int q, int32_t* iters, int32_t* loads, void* stream);

/*
 * Token placement for dispatch and the grouped GEMM's work list.
 *   slot_base [G,E,G] int32: buffer row of the first token of bucket (g,e,d)
 *   segs [cap,4] int32 {row_start, nrows, wslot, expert} in plan order, n_seg [1], mtile_prefix [cap+1]
 *   fetch [E] int32: experts this rank must fetch (non-resident with work), plan order; n_fetch [1]
 * LOCAL: segments are (dest, expert) over the whole [G] buffer, wslot = expert.
 * EP:    segments are (expert, source) of rank `me`'s receive buffer; wslot = index of the expert
 *        among me's home experts (ascending id), fetched experts get slots n_home + fetch ordinal,
 *        or n_home + (ordinal % cache_slots) with a bounded cache (cache_slots > 0): fetch i then
 *        reuses the slot of fetch i - cache_slots, the first to free up (engine.py:239-257).
 * cap >= G*E.
 */
HM_API int hm_dispatch_layout(const int32_t* S, const int32_t* home, int G, int E, int mode, int me, int32_t* slot_base,
                       int32_t* segs, int32_t* n_seg, int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch,
                       int cache_slots, void* stream);

/*
 * Fused planner: the whole step-2/3 stage in one single-CTA launch (histogram reduce ->
 * hm_schedule -> hm_dispatch_layout).  Either tile_hist (+ tiles_per_rank; LOCAL layout, G ranks
 * on this device: also writes m_all_out [G,E] and tile_off) or m_all_in [G,E] (EP: after the
 * metadata all_gather) is given.  Outputs as hm_schedule + hm_dispatch_layout.
 * Requires (E + 4*G*E + G*E*G + 3*E) * 4 bytes <= 200 KB.
 */
HM_API int hm_plan(const int32_t* tile_hist, int tiles_per_rank, const int32_t* m_all_in, const int32_t* home, int G,
                   int E, int q, int rebalance, int mode, int me, int32_t* m_all_out, int32_t* tile_off, int32_t* S,
                   int32_t* iters, int32_t* loads, int32_t* slot_base, int32_t* segs, int32_t* n_seg,
                   int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch, int cache_slots, void* stream);

/*
 * Scatter (K4): copy token rows to their scheduled buffer rows (one read of x, k 128-bit-vector
 * writes).  Token t's source rank is src_rank_base + t / tokens_per_rank; its r-th assignment to
 * expert e goes to the first dest d with cumsum_d S[src,e,d] > r (split-bucket contract).
 *   out [rows, d] bf16, pos [T, k] int32 (row index of each assignment in `out`),
 *   inv [rows] int32 or NULL: inverse map, inv[pos[t,j]] = t*k + j (lets the FFN2 epilogue write
 *   its rows token-major so the combine streams contiguous memory).
 *   out == NULL: index-only scatter (pos + inv, no row copies); the FFN1 GEMM then gathers the
 *   rows itself (hm_grouped_gemm a_gather = inv, a_gather_div = k).
 */
HM_API int hm_permute(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
               const int32_t* S, const int32_t* slot_base, int n_ranks, int tokens_per_rank, int src_rank_base,
               int G, int E, int k, int d, void* out, int32_t* pos, int32_t* inv, void* stream);

/*
 * K6 fetch pairs inside a grouped-GEMM launch (bounded expert cache, engine.py:204-275).
 * The last `pairs` CTA pairs of the launch copy experts instead of computing, so the copy and the
 * GEMM tiles it gates - and the GEMM tiles whose completion frees the cache slots - are
 * co-resident by construction (no cross-stream dependency).  Fetch i goes to slot
 * first_slot + i % n_slots and, for i >= n_slots, only after the launch's slot_done count of
 * expert fetch[i - n_slots] reaches 16 x its pair tiles (its occupant is finished).
 *   phase 1 (FFN1 launch): every expert's gate/up block (src_in -> dst_in, ready_in), then the
 *                          down blocks of the first min(n_slots, *n_fetch) (src_out -> dst_out)
 *   phase 2 (FFN2 launch): the remaining down blocks, gated by FFN2's own slot_done counts
 * Copies are TMA bulk transfers global -> shared -> global (32 KB chunks, 6 in flight per CTA).
 */
typedef struct hm_fetch_plan {
  const int32_t* fetch;     /* [E] experts to fetch in plan order (the layout's fetch list) */
  const int32_t* n_fetch;   /* [1] */
  const uint64_t* src_in;   /* [E] device pointer of expert e's gate/up (or W1) block */
  const uint64_t* src_out;  /* [E] device pointer of expert e's down (W2) block */
  void* dst_in;             /* slot s of the gate/up cache at dst_in + s * in_bytes */
  void* dst_out;            /* slot s of the down cache at dst_out + s * out_bytes */
  uint64_t in_bytes;
  uint64_t out_bytes;
  int32_t first_slot;
  int32_t n_slots;
  int32_t* ready_in;        /* [E] per-expert flags set to `value` */
  int32_t* ready_out;
  int32_t* counters;        /* scratch, n_counters >= 2 * E, zeroed by the launch */
  int32_t n_counters;
  int32_t value;
  int32_t pairs;            /* fetch pairs (>= 1) */
  int32_t phase;            /* 1 or 2 */
} hm_fetch_plan;

/*
 * Grouped expert GEMM (K5), tcgen05/TMEM/TMA: for every segment, out[rows] = epi(A[rows] W[wslot]^T).
 *   A [a_rows, K] bf16; W [w_rows, K] bf16 with w_rows = slots*N; out [a_rows, N] (or N/2 for SWIGLU).
 *   row_map [rows] int32 or NULL: output row of buffer row r is row_map[r] (scatter epilogue).
 *   a_gather [rows] int32 or NULL: fused scatter - buffer row r reads A row a_gather[r] / a_gather_div
 *   (TMA tile::gather4 straight from the token activations; with the inverse permutation of
 *   hm_permute and div = k this is the token of each assignment).  A is then [a_rows, K].
 *   slot_ready [E] int32 or NULL: tiles of a segment whose weight slot is >= ready_from_slot (a
 *   fetched expert, K6) wait until slot_ready[expert] >= epoch (per expert, not per slot: a
 *   bounded cache reuses slots within one forward, engine.py:239-257).
 *   slot_done [E] int32 or NULL: every epilogue warp (16 per 256-row pair tile) adds 1 to
 *   slot_done[expert] when it has finished a tile of a fetched expert (release) - the K6 channel
 *   overwrites that expert's cache slot once the count reaches 16 x its pair tiles.
 *   fetch: NULL, or the K6 fetch pairs of this launch (hm_fetch_plan; needs slot_done).
 * Requires N % 256 == 0, K % 64 == 0.
 */
HM_API int hm_grouped_gemm(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K, const int32_t* segs,
                    const int32_t* n_seg, const int32_t* mtile_prefix, int epilogue, void* out, const int32_t* row_map,
                    const int32_t* a_gather, int a_gather_div, const int32_t* slot_ready, int ready_from_slot,
                    int epoch, int32_t* slot_done, const hm_fetch_plan* fetch, void* stream);

/*
 * Swap-AB grouped GEMM for weight-streaming shapes (tens of rows per expert, e.g. Switch top-1):
 * the MMA's M is 256 weight rows and N 64 token rows, so a small expert pads to 64 token rows
 * instead of 128-256 rows of A.  A [a_rows, K] bf16 (no gather), W [slots*N, K]; epilogue
 * HM_EPI_RELU or HM_EPI_STORE; out [a_rows(or row_map target), N] row r (-> row_map[r]).
 * y != NULL (STORE, top-1 combine): y[row_map[r]] = (residual +) topk_w[row_map[r]] * row, the
 * arithmetic of hm_combine with k = 1 (bit-identical); out is then not written (may be NULL).
 * At most 512 segments.  Same outputs as hm_grouped_gemm (fp32 accumulation over K in order).
 */
HM_API int hm_grouped_gemm_swap(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                                const int32_t* segs, const int32_t* n_seg, int epilogue, void* out,
                                const int32_t* row_map, const float* topk_w, const void* residual, void* y,
                                void* stream);

/*
 * FFN2 with the weighted combine (K7) fused into its epilogue (LOCAL layout, Alg. 1 steps 5-6,
 * PAPER.md:613-616): the STORE epilogue scatters expert row r to Y row row_map[r] = t*k + j as
 * hm_grouped_gemm does, and the k-th arriving row of every (token t, 64-column chunk) computes
 *   y[t, chunk] = (residual[t, chunk] +) sum_{j<k} topk_w[t, j] * Y[t*k + j, chunk]
 * in fp32 in slot order - bit-identical to hm_combine(Y, NULL, topk_w, ...) after hm_grouped_gemm.
 *   counters [T * N/64] uint32, zero before the first call; every call leaves them zero again.
 *   k == 1 (top-1, Switch): the epilogue writes y[t] = (residual[t] +) w[t] * Y_row directly (same
 *   arithmetic, bit-identical); Y is not written and may be NULL, counters may be NULL.
 *   residual [T, N] bf16 or NULL; y [T, N] bf16.  Requires 1 <= k <= 32.
 */
HM_API int hm_grouped_gemm_combine(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                                   const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix, void* Y,
                                   const int32_t* row_map, const float* topk_w, int k, const void* residual, void* y,
                                   uint32_t* counters, void* stream);

/*
 * Async expert fetch (K6): copy `bytes` from src (peer HBM through UVA/NVLink, or pinned host
 * memory) into dst on `stream` (the dedicated fetch stream), then publish *ready_flag = epoch.
 */
HM_API int hm_fetch_expert(void* dst, const void* src, size_t bytes, int32_t* ready_flag, int epoch, void* stream);

/*
 * Peer-HBM access for K6 over NVLink/NVSwitch: export a device allocation as a 64-byte CUDA IPC
 * handle (host buffer), open a peer's handle in this process, close it.  The expert-parallel
 * layer exchanges handles once at setup so every rank can fetch any home expert directly.
 */
HM_API int hm_ipc_get_handle(const void* dev_ptr, void* handle_out /* 64 B, host */,
                             size_t* offset_out /* dev_ptr - allocation base, or NULL */);
HM_API int hm_ipc_open(const void* handle /* 64 B, host */, void** dev_ptr_out);
HM_API int hm_ipc_close(void* dev_ptr);

/*
 * Combine (K7): y[t] = sum_j w[t,j] * Y[pos[t,j]] in fp32, slots in order j = 0..k-1, bf16 out.
 * pos == NULL means Y is token-major [T*k, d] (row t*k + j), the layout the FFN2 epilogue writes
 * through row_map.  residual [T, d] bf16 or NULL: decoder residual fused in, the fp32
 * accumulation starts from it (y = x + sum_j w Y_j).
 */
HM_API int hm_combine(const void* Y, const int32_t* pos, const float* topk_w, int T, int k, int d,
                      const void* residual, void* y, void* stream);

/* ------------------------------------------------------------------------------------------
 * Expert parallelism over NVSwitch peer memory (ep.py transport "p2p"): every rank's receive
 * buffer, token-index buffer, output buffer and flags are mapped into every other rank once
 * (hm_ipc_*); the replicated schedule S then places every row without any host round trip
 * (SURVEY.md §8(e)).  Replaces the NCCL all_to_all pair of engine.py:342-375 / PAPER.md:606-616.
 * ---------------------------------------------------------------------------------------- */

/*
 * From S [G,E,G]: dst_delta[d] = row of this rank's assignments in d's receive buffer minus their
 * row in the send layout of hm_dispatch_layout (HM_LAYOUT_EP), and recv_split [G+1] = first
 * receive row of each source (flows of engine._exchange_byte_vectors, engine.py:278-284).
 */
HM_API int hm_ep_offsets(const int32_t* S, int G, int E, int me, int32_t* dst_delta, int32_t* recv_split,
                         void* stream);

/*
 * Fused scatter + dispatch (Alg.1 step 4 + the all_to_all): token row t is read once and
 * stored into dst_rows[d] (receive buffer of destination rank d, a peer pointer) at its
 * receive row, and t*k + j into dst_tok[d] at the same row.  dst_rows / dst_tok: device arrays
 * of G pointers.  pos [T*k] (or NULL) gets the send-layout row, as hm_permute would.
 * dst_delta == NULL: slot_base is an HM_LAYOUT_EP_EXPERT layout (rows of every destination's
 * expert-major buffer, no send layout), and the token index stored is (me << 24) | (t*k + j) so
 * the receiver's FFN2 can route each row home (hm_grouped_gemm_remote with out_split == NULL).
 */
HM_API int hm_dispatch_push(const void* x, const int32_t* topk_idx, const int32_t* lrank, const int32_t* tile_off,
                            const int32_t* S, const int32_t* slot_base, const int32_t* dst_delta, int tokens, int me,
                            int G, int E, int k, int d, const uint64_t* dst_rows, const uint64_t* dst_tok,
                            int32_t* pos, void* stream);

/*
 * Expert-ordered dispatch (EP p2p, overlapped with FFN1).  hm_plan_dispatch is hm_plan with
 * m_all_in and the HM_LAYOUT_EP_EXPERT layout of rank `me`, plus this rank's push work list:
 *   push_items [G*E, 4] int32: item v = p*G + d is me's bucket of the expert at position p of
 *     destination d's plan order (engine.py:233-234): (expert, first rank among me's assignments
 *     to it, rows, first row in d's receive buffer); rows 0 where d has fewer than p+1 experts;
 *   push_cprefix [G*E + 1]: exclusive prefix of 8-row units per item (-1 at [G*E] if the batch
 *     left the planner's fast path: >= 2^21 assignments, which the push then reports by trapping);
 *   push_ebase [E + 1]: exclusive prefix of m_all[me] over experts.
 * Requires a power-of-two G and a harmony / static policy.
 * hm_dispatch_push_ordered copies the rows unit by unit in that order (8 rows of one bucket per
 * unit, one warp each) into dst_rows[d] / tags dst_tok[d] as hm_dispatch_push with dst_delta == NULL does, and
 * after each unit adds its row count to ((int32_t*)dst_arrive[d])[expert] (system-scope release).
 * order [tokens*k] int32 scratch; pos [tokens*k] or NULL as hm_dispatch_push; sync [2] uint32
 * scratch (zeroed by the call).  One CTA per SM with a grid barrier: launch it right before the
 * FFN1 that consumes it, nothing else running on the device's SMs in between.
 * hm_grouped_gemm_arrive is hm_grouped_gemm (TMA-loaded A, no row map) whose producers wait per
 * segment until a_arrive[expert] >= the segment's rows (system-scope acquire); pdl = 1 launches
 * it with programmatic stream serialisation so it starts while the push kernel before it in the
 * stream still runs (it completes only after that kernel has).
 */
HM_API int hm_plan_dispatch(const int32_t* m_all_in, const int32_t* home, int G, int E, int q, int rebalance, int me,
                            int32_t* S, int32_t* iters, int32_t* loads, int32_t* slot_base, int32_t* segs,
                            int32_t* n_seg, int32_t* mtile_prefix, int32_t* fetch, int32_t* n_fetch, int cache_slots,
                            int32_t* push_items, int32_t* push_cprefix, int32_t* push_ebase, void* stream);
HM_API int hm_dispatch_push_ordered(const void* x, const int32_t* topk_idx, const int32_t* lrank,
                                    const int32_t* tile_off, const int32_t* S, const int32_t* slot_base,
                                    const int32_t* push_items, const int32_t* push_cprefix, const int32_t* push_ebase,
                                    int tokens, int me, int G, int E, int k, int d, const uint64_t* dst_rows,
                                    const uint64_t* dst_tok, const uint64_t* dst_arrive, int32_t* order, int32_t* pos,
                                    uint32_t* sync, void* stream);
HM_API int hm_grouped_gemm_arrive(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                                  const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix,
                                  int epilogue, void* out, const int32_t* slot_ready, int ready_from_slot, int epoch,
                                  int32_t* slot_done, const hm_fetch_plan* fetch, const int32_t* a_arrive, int pdl,
                                  void* stream);

/*
 * hm_grouped_gemm whose output rows go to other ranks (FFN2 + the return all_to_all): the rows
 * of a segment starting at receive row r0 belong to source g with out_split[g] <= r0 <
 * out_split[g+1], and land in out_ptrs[g] (device array of n_out peer pointers) at row
 * row_map[r].  out_split == NULL (expert-major receive buffer): row r lands in
 * out_ptrs[row_map[r] >> 24] at row row_map[r] & 0xFFFFFF.  2-CTA kernel only.
 */
HM_API int hm_grouped_gemm_remote(const void* A, int64_t a_rows, const void* W, int64_t w_rows, int N, int K,
                                  const int32_t* segs, const int32_t* n_seg, const int32_t* mtile_prefix,
                                  int epilogue, const uint64_t* out_ptrs, const int32_t* out_split, int n_out,
                                  const int32_t* row_map, const int32_t* slot_ready, int ready_from_slot, int epoch,
                                  int32_t* slot_done, const hm_fetch_plan* fetch, void* stream);

/*
 * Device-driven K6 (engine.py:253-265): copy expert fetch[i] (i < *n_fetch, plan order, from the
 * layout's fetch list) from src_in[e] / src_out[e] (device arrays of E pointers: the home rank's
 * HBM through IPC, or pinned host memory) into cache slot first_slot + i of dst_in / dst_out
 * (slot strides in_bytes / out_bytes), publishing ready_in / ready_out[e] = value (per EXPERT)
 * as each block lands.  counters [n_counters >= 2 * *n_fetch] int32 scratch (zeroed by the call);
 * ctas <= 0: default.  *n_fetch > n_slots traps the launch (never a silent truncation): a bounded
 * cache is fetched inside the GEMM launches (hm_fetch_plan).
 */
HM_API int hm_fetch_experts(const int32_t* fetch, const int32_t* n_fetch, const uint64_t* src_in,
                            const uint64_t* src_out, size_t in_bytes, size_t out_bytes, void* dst_in, void* dst_out,
                            int first_slot, int n_slots, int32_t* ready_in, int32_t* ready_out, int32_t* counters,
                            int n_counters, int value, int ctas, void* stream);

/*
 * Stream-ordered flags: hm_stream_signal writes `value` to each of n device addresses
 * (flags: HOST array of device pointers, typically peers' flag words) after all prior work
 * on the stream, with a system-scope fence; hm_stream_wait blocks the stream until each of the
 * n consecutive int32 at `flags` is >= value.  Neither occupies an SM.
 */
HM_API int hm_stream_signal(void* const* flags, int n, uint32_t value, void* stream);
HM_API int hm_stream_wait(const int32_t* flags, int n, uint32_t value, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HARMOE_H_ */
