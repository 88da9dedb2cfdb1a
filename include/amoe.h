/*
 * amoe.h — C ABI of libamoe, the B200 (sm_100a) hot path of Asynchronous Expert Parallelism
 * (AEP), arXiv 2505.08944 "Toward Cost-Efficient Serving of Mixture-of-Experts with Asynchrony".
 *
 * The calls follow the paper's statement of the expert-side execution engine (§3.2,
 * L220-L236, Fig. "engine"):
 *   amoe_enqueue   receptor/dispatcher: route a token (top-K, L227) and put each of its K
 *                  duplicated legs into the µ-queue of (layer, expert) on the GPU hosting that
 *                  expert (L221 "segregates ... by the LayerID", L236 "permutes tokens by
 *                  expert ID ... sent to appropriate expert workers").
 *   amoe_pick      scheduler: Algorithm 1 "Defragging Scheduler" (L266-L295), MTFS (L262),
 *                  FLFS (L264) over a queue-depth snapshot (host C++, plumbing).
 *   amoe_rebatch   executor: drain the selected µ-queue(s) "just in time" into one contiguous
 *                  input batch (L75, L222 "our custom CUDA kernel for preparing a contiguous
 *                  input token batch from many individually arrived token batches").
 *   amoe_expert_ffn executor: run the expert layer (SwiGLU gate/up/down) over that batch.
 *   amoe_forward   dispatcher: send every output row back to its token's home (attention-DP)
 *                  rank (L236 "permuted by their assigned attention DP rank") — here a one-sided
 *                  NVLink store into the home's token pool, replacing the two-phase
 *                  ZeroMQ + NCCL transfer (L303-L320).
 *   amoe_combine   token pool + top-K merge (L228, L175): when all K legs of a token arrived,
 *                  h += Σ_k w_k·O_k, x = rmsnorm(h), relabel to layer+1 (L209, L236) and
 *                  enqueue it there (fused amoe_enqueue), or retire it after the last pass.
 *
 * CONVENTIONS (apply to every call)
 *  - Ownership: the caller allocates ALL device memory (workspace, weights, router table,
 *    group buffers) and keeps it alive while the context uses it. The library only borrows
 *    pointers; it never allocates or frees device memory. Host arrays are copied on entry.
 *  - Pointers marked "device" are CUDA device pointers on the context's current device;
 *    "host" pointers are ordinary host memory (pinned memory recommended for *_host calls).
 *  - Asynchrony: calls taking a cudaStream_t (passed as void*) enqueue work on that stream and
 *    return immediately, except where "synchronises" is stated.
 *  - Errors: host-detectable errors return synchronously (AMOE_EINVAL, AMOE_ENOTHOSTED,
 *    AMOE_ECUDA ...). Device-side invariant breaches (ring overflow, leg count > K, expert
 *    index out of range, leg for a non-hosted queue) are latched into a device error word and
 *    reported as AMOE_EDEVICE by amoe_check() / amoe_run(); amoe_error_info() gives details.
 *  - Contexts: one per (process, GPU, rank); not thread-safe. Issue a context's launches on one
 *    stream at a time (its FFN tile-claim counters and group scratch live in the workspace).
 *  - Launches use programmatic dependent launch (kernel boundaries on a stream overlap the next
 *    kernel's launch with the previous kernel's tail); AMOE_PDL=0 turns it off.
 *  - Empty work is legal: draining empty queues yields n = 0 and the later calls are no-ops.
 *  - Layouts are row-major; bf16 is IEEE bfloat16 bit patterns (uint16), fp32 is float.
 */
#ifndef AMOE_H
#define AMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMOE_MAX_G 8          /* GPUs in one NVSwitch box */
#define AMOE_MAX_E 256        /* routed experts per layer */
#define AMOE_MAX_GROUP 128    /* queues drained/executed by one grouped launch */

typedef enum amoe_status {
  AMOE_OK = 0,
  AMOE_IDLE = 1,        /* amoe_pick: every hosted queue is empty */
  AMOE_EINVAL = 2,      /* bad argument / unsupported shape */
  AMOE_ENOTHOSTED = 3,  /* (layer, expert) is not hosted by this rank */
  AMOE_ECUDA = 4,       /* a CUDA runtime call failed */
  AMOE_EDEVICE = 5,     /* latched device-side invariant breach */
  AMOE_EPEER = 6,       /* peer workspaces missing or inconsistent */
  AMOE_ENOMEM = 7       /* workspace smaller than amoe_workspace_bytes() */
} amoe_status;

/* Opaque per-(process, GPU, rank) context; host memory owned by the library. */
typedef struct amoe_ctx amoe_ctx;
typedef amoe_ctx* amoe_ctx_t;

typedef enum amoe_dtype { AMOE_BF16 = 0, AMOE_FP32 = 1 } amoe_dtype;
/* AMOE_SYNC is the synchronous expert-parallel baseline on the same kernels (SURVEY.md §8(f) f1,
 * PAPER.md L65-L66, L123): layers run in lockstep; a rank takes layer l+1 only after every rank's
 * homed tokens have merged layer l (a box-wide barrier per layer, flags stored into every peer's
 * workspace), which is the dependency an all-to-all before and after each expert layer imposes.
 * Every admitted token must start at the layer of this rank's last amoe_enqueue call. */
/* AMOE_DEFRAG_GLOBAL is Algorithm 1 with a box-wide lookahead (PAPER.md
 * L266-L297 read with Q[l, g] = tokens of layer l on every GPU g, DESIGN.md c11): the picked queue's
 * own term is this GPU's depth, the lookahead term of block b' sums b' over every rank's queues,
 * read from the peers' queue counters over NVLink (amoe_run only; identical to AMOE_DEFRAG at G = 1). */
typedef enum amoe_policy {
  AMOE_DEFRAG = 0,
  AMOE_MTFS = 1,
  AMOE_FLFS = 2,
  AMOE_SYNC = 3,
  AMOE_DEFRAG_GLOBAL = 4
} amoe_policy;

/* Model / placement configuration. */
typedef struct amoe_config {
  int32_t L;           /* expert layers (decoding blocks) */
  int32_t E;           /* routed experts per layer, <= AMOE_MAX_E */
  int32_t K;           /* top-K, 1 <= K <= 8, K <= E */
  int32_t S;           /* shared experts per layer (weight 1, run on the token's home), <= 4 */
  int32_t d;           /* model width, multiple of 128 */
  int32_t ff;          /* expert FFN width, multiple of 128 */
  int32_t G;           /* GPUs (ranks) in the box, 1..AMOE_MAX_G */
  int32_t rank;        /* this rank */
  int32_t T_slots;     /* token slots homed on each rank */
  int32_t dtype;       /* amoe_dtype: BF16 (tensor cores) or FP32 (exact-reference mode) */
  int32_t max_batch;   /* cap on tokens drained from one queue per pick; 0 = drain all */
  int32_t rows_cap;    /* rows of the internal group scratch used by amoe_run; 0 = default */
  float rms_eps;       /* RMSNorm epsilon; 0 -> 1e-6 */
  int32_t owner[AMOE_MAX_E];  /* owner[e] = rank hosting expert e for all layers (PAPER.md
                                 L240); all-zero with G > 1 means the default e mod G */
} amoe_config;

/* One µ-queue entry: a duplicated token leg (Table 1 metadata subset). 16 bytes.
 * token_slot = RequestID role (slot on the home rank), home = attention-DP rank, k = which of
 * the K legs (K..K+S-1 for shared experts), w = Topk_weight, seq = ring position + 1 (written
 * last; the consumer only takes a contiguous published prefix). */
typedef struct amoe_leg {
  int32_t token_slot;
  int16_t k;
  int16_t home;
  float w;
  uint32_t seq;
} amoe_leg;

/* Buffers of one grouped execution (caller-owned device memory). rows_cap rows each. */
typedef struct amoe_group {
  int32_t nq;                        /* queues in the group, 1..AMOE_MAX_GROUP */
  int32_t layer[AMOE_MAX_GROUP];     /* (layer, expert) of each queue; expert >= E = shared */
  int32_t expert[AMOE_MAX_GROUP];
  int32_t rows_cap;                  /* rows in tile / meta / act / out */
  void* tile;                        /* device [rows_cap, d] storage dtype: drained inputs */
  amoe_leg* meta;                    /* device [rows_cap]: the drained legs, row-aligned */
  int32_t* qinfo;                    /* device [3 * AMOE_MAX_GROUP]: n[q], row_off[q], start[q] */
  void* act;                         /* device [rows_cap, ff]: SwiGLU activations */
  void* out;                         /* device [rows_cap, d]: expert outputs */
  int32_t max_rows_hint;             /* largest queue length expected (0 = unknown), a
                                        performance hint: <= 128 selects the 1-CTA (M = 128)
                                        FFN kernels, which stream cold-expert weights faster;
                                        any n remains correct */
} amoe_group;

typedef struct amoe_run_params {
  int32_t policy;      /* amoe_policy */
  int32_t W;           /* Algorithm 1 lookahead depth (reading c11), default 4 */
  float delta;         /* Algorithm 1 weight decay δ, default 0.5 */
  int32_t grouped;     /* 1: one launch runs every nonempty hosted queue of the picked layer */
  int32_t max_picks;   /* 0: run until every token retired (all ranks). > 0 (single rank):
                          stepping mode for open-loop serving — return after this many picks or
                          as soon as nothing is runnable; the caller admits new tokens between
                          calls (amoe_token_init + amoe_enqueue) */
} amoe_run_params;

typedef struct amoe_run_stats {
  int64_t picks;           /* scheduler decisions (grouped launches) */
  int64_t queues_run;      /* (layer, expert) executions */
  int64_t legs;            /* legs executed on this rank */
  int64_t token_layers;    /* merges completed on this rank (homed tokens) */
  int64_t kernel_launches; /* libamoe kernels launched */
  int64_t idle_polls;      /* scheduler polls that found nothing to run */
  int64_t idle_ns;         /* host wall time of those polls, counted from the moment the poll's
                              stream synchronisation returned (this rank's earlier kernels done)
                              to the next poll: the GPU had nothing of this rank's queues to run
                              = stall (includes AMOE_GROW_WAIT deferrals) */
  int64_t wall_ns;         /* host wall time of the whole amoe_run call */
  int64_t barriers;        /* AMOE_SYNC: layer barriers passed */
} amoe_run_stats;

/* ---- context ------------------------------------------------------------------------ */

/* Bytes of device workspace this rank needs (rings, token state, pools, counters, tensor-map
 * table, group scratch for amoe_run). Same value on every rank (symmetric layout). 0 = bad cfg. */
size_t amoe_workspace_bytes(const amoe_config* cfg);

/* Create a context over caller-allocated `workspace` (device, >= amoe_workspace_bytes, 256-B
 * aligned). Zeroes counters and token state with a synchronous cudaMemset. cfg copied. */
amoe_status amoe_create(const amoe_config* cfg, void* workspace, size_t bytes, amoe_ctx_t* out);

/* Register every rank's workspace base (host array [G] of device addresses valid in THIS
 * process: opened CUDA IPC handles / symm_mem buffer_ptrs, or local aliases for loopback tests).
 * peer_ws[rank] must equal this context's workspace. Setup only. The caller must synchronise all
 * ranks (device sync + process barrier) after every rank's amoe_create and before the first
 * amoe_enqueue anywhere: amoe_create zeroes the rings that peers push legs into. Workspaces on
 * other devices get peer access enabled from the current device (cudaDeviceEnablePeerAccess).
 * Errors: AMOE_EPEER if an address is null, unaligned, not a device address, or on a device
 * this one cannot reach as a peer. */
amoe_status amoe_import_peers(amoe_ctx_t ctx, const uint64_t* peer_ws, int G);

/* Register expert weights of (layer, expert) hosted here (expert >= E: shared expert
 * expert-E, hosted on every rank). w1 (gate) and w3 (up): device [ff, d]; w2 (down): device
 * [d, ff]; storage dtype, row-major (K-major operands). Borrowed. Builds the TMA descriptors
 * once (bf16). ENOTHOSTED if owner[expert] != rank. Synchronous (small H2D copy). */
amoe_status amoe_set_expert(amoe_ctx_t ctx, int layer, int expert, const void* w1, const void* w3,
                            const void* w2);

/* Router logits used when amoe_combine relabels a token to its next layer (the paper's eval
 * replaces the gate by random routing from a fitted distribution): device fp32
 * [n_tables][L][T_slots][E]; a token at (pass p, layer l) uses table p mod n_tables. */
amoe_status amoe_set_router(amoe_ctx_t ctx, const float* table, int n_tables);

/* Router gate of `layer` (the gate is the last op of the attention layer,
 * PAPER.md L175, L227): logits z[e] = Σ_j x[j]·wg[e][j] (+ bias[e]), fp32 accumulation, on the
 * token's x = rmsnorm(h) at that layer, then the same top-K + softmax as table routing. wg:
 * device [E][d] storage dtype, row-major; bias: device fp32 [E] or NULL. Borrowed. A layer with
 * a gate routes with it (in amoe_combine, and in amoe_enqueue when logits and topk_* are NULL);
 * other layers use the router table. wg = NULL clears the layer's gate. EINVAL when d exceeds
 * 4096 (bf16) / 2048 (fp32). Synchronous (16-byte H2D copy). */
amoe_status amoe_set_gate(amoe_ctx_t ctx, int layer, const void* wg, const float* bias);

/* Checked mode (schedule replay): every drain (amoe_rebatch and the
 * drains inside amoe_run's launches) appends, per nonempty queue it drained, an execution record
 * and a copy of the legs it took, in FIFO order, to `buf` (device, caller-owned, 16-B aligned;
 * NULL turns logging off). Layout, uint32 words: [0] executions logged, [1] legs logged,
 * [2] record capacity, [3] leg capacity (both set here from `bytes`), [4..8) reserved; then
 * records {qid = layer * H + local queue, start = ring position of the first drained leg, n,
 * offset of its first leg} x capacity; then amoe_leg x capacity, with `seq` replaced by the
 * token's pass. Counts beyond capacity are counted, not written. Slows drains (one CTA copies
 * the legs): tests only. Synchronises the device. */
amoe_status amoe_set_exec_log(amoe_ctx_t ctx, void* buf, size_t bytes);

/* Admit tokens: for i < T, slot = slots[i] (device int32): h[slot] = h0[i] (device [T, d]
 * storage dtype), x[slot] = rmsnorm(h0[i]), pass = pass, layer = 0, pool cleared. */
amoe_status amoe_token_init(amoe_ctx_t ctx, const int32_t* slots, int T, const void* h0, int pass,
                            void* stream);

/* a1 + a2: route tokens slots[0..T) (device int32, homed here, x already set) at `layer` and
 * put their legs into the µ-queues of the owners (local store or NVLink peer store + remote
 * atomic reservation). Routing either from logits (device fp32 [T, E]: top-K, ties to the lower
 * expert, softmax over the K selected) or given topk_idx/topk_w (device [T, K]) when logits is
 * NULL. The chosen idx/w are kept in the token state (amoe_get_buffer AMOE_BUF_TOK_IDX/W). */
amoe_status amoe_enqueue(amoe_ctx_t ctx, int layer, const int32_t* slots, int T, const float* logits,
                         const int32_t* topk_idx, const float* topk_w, void* stream);

/* Queue-depth snapshot Q[l][q] = published - drained, host out [L * H] (H = amoe_hosted()),
 * column q = local queue index (see amoe_local_queue). Synchronises `stream`. */
amoe_status amoe_queue_depths(amoe_ctx_t ctx, uint32_t* host_out, void* stream);

/* Top-1 direct forwarding (PAPER.md L463 — with one expert per token there is
 * no top-K merge to wait for; L227-L228 — a token ready by itself skips the token pool): when on,
 * amoe_run's executing rank merges each token it ran (h += w·O, the combine's arithmetic),
 * normalises it, routes its next layer and scatters the next leg straight into that expert's queue;
 * the home's pool, leg counter, combine ring and combine launch are not used. Requires K == 1 and
 * S == 0 (EINVAL otherwise); at G > 1 every layer must route with a gate (amoe_set_gate, checked
 * by amoe_run: EINVAL). Results equal the pooled path bit for bit. */
amoe_status amoe_set_direct(amoe_ctx_t ctx, int on);

/* Box-wide depth per block (the AMOE_DEFRAG_GLOBAL lookahead input): host out [L], entry l = queued
 * legs of layer l summed over every rank's queues, read on device from the peers' queue counters
 * (amoe_import_peers first when G > 1; EPEER otherwise). Synchronises `stream`. */
amoe_status amoe_box_depths(amoe_ctx_t ctx, uint32_t* host_out, void* stream);

/* Algorithm 1 / MTFS / FLFS over a host snapshot Q [L * H] (W = lookahead depth, δ = decay;
 * the lookahead divisor N_E is the block's expert count E + S, routed plus shared, box-wide —
 * DESIGN.md reading c11; ties to the smallest (layer, queue)). AMOE_IDLE when all empty.
 * AMOE_DEFRAG_GLOBAL is not accepted here (it needs the peers' counters: amoe_run only). */
amoe_status amoe_pick(amoe_ctx_t ctx, const uint32_t* Q, int policy, int W, float delta, int* layer,
                      int* queue);

/* Context-free form of amoe_pick (pure host code): Q [n_blocks * n_queues], divisor n_experts.
 * Returns AMOE_OK with *block/*queue set, AMOE_IDLE when all empty, AMOE_EINVAL on bad args. */
amoe_status amoe_schedule(const uint32_t* Q, int n_blocks, int n_queues, int n_experts, int policy, int W,
                          float delta, int* block, int* queue);

/* Algorithm 1 with an explicit lookahead (the AMOE_DEFRAG_GLOBAL pick, pure host code): Q_local
 * [n_blocks * n_queues] = this GPU's hosted depths (the candidates, L283-L286); block_totals
 * [n_blocks] = queued legs of each block summed over EVERY GPU's queues (the lookahead of
 * L277-L280), divisor n_experts. AMOE_OK / AMOE_IDLE (every local queue empty) / AMOE_EINVAL. */
amoe_status amoe_schedule_global(const uint32_t* Q_local, const uint32_t* block_totals, int n_blocks,
                                 int n_queues, int n_experts, int W, float delta, int* block, int* queue);

/* a4: drain up to max_tokens (0 = all published, also capped by cfg.max_batch and rows_cap)
 * FIFO entries of each queue of `grp` into grp->tile rows (queue q at rows row_off[q] ..
 * row_off[q]+n[q]-1, row_off a multiple of 128), grp->meta = the drained legs. Pulls each
 * token's x row from its home (local or NVLink peer load). qinfo written on device. */
amoe_status amoe_rebatch(amoe_ctx_t ctx, const amoe_group* grp, int max_tokens, void* stream);

/* a5 + a6: out[r] = W2 (silu(W1 tile[r]) ⊙ W3 tile[r]) for every drained row of every queue of
 * grp; act holds the bf16 SwiGLU activations. bf16: tcgen05/TMEM tensor-core kernels;
 * fp32: exact SIMT kernels. Rows beyond n[q] are not written. */
amoe_status amoe_expert_ffn(amoe_ctx_t ctx, const amoe_group* grp, void* stream);

/* a5 + a6 + a7 fused (what amoe_run uses): as amoe_expert_ffn, but the down-GEMM epilogue stores
 * each output row directly into its token's home pool (NVLink peer store when remote) and
 * counts it on the token's leg counter in 128-column pieces; grp->out is not written. The fp32
 * mode runs amoe_expert_ffn then the amoe_forward kernel. */
amoe_status amoe_expert_ffn_forward(amoe_ctx_t ctx, const amoe_group* grp, void* stream);

/* a4 + a5 + a6 + a7 fused (what amoe_run uses): drain the group's queues, then the expert FFN
 * with the re-batch gather inside the gate/up GEMM's A-operand load (TMA tile::gather4 of the
 * tokens' x rows by slot; the drained legs are read from the rings) and the forward inside the
 * down GEMM's epilogue. grp->tile/meta/out are not written. Single GPU, bf16; otherwise it runs
 * amoe_rebatch + amoe_expert_ffn_forward. */
amoe_status amoe_rebatch_ffn_forward(amoe_ctx_t ctx, const amoe_group* grp, int max_tokens, void* stream);

/* a4 + a5 + a6 + a7 of a COLD pick in ONE launch (small
 * batches are weight-streaming bound): queue q of `grp` drains exactly n[q] legs (0..128) from ring
 * position start[q] — the queue's consumer head, as a queue-depth snapshot gives it with
 * n[q] <= its published depth (the scheduler's decision) — gathers their x rows,
 * runs the SwiGLU expert and stores every output row into its home's token pool (a7). Writes
 * grp->qinfo (n, row offset, start); uses grp->act ([nq * n_pad, ff], n_pad = max n rounded up
 * to 16). bf16 contexts with d % 256 == 0 only (EINVAL otherwise). A head that is not start[q] latches device fault
 * 12 (queue, start, head); an entry never published traps after 4 s (ECUDA). */
amoe_status amoe_execute_cold(amoe_ctx_t ctx, const amoe_group* grp, const uint32_t* start, const int32_t* n,
                              void* stream);

/* a7 (return leg): store out rows into pool[home][token_slot][k] (NVLink store when remote),
 * bump the token's leg counter (release, system scope); the leg completing K (+S) appends the
 * token to its home's combine ring. */
amoe_status amoe_forward(amoe_ctx_t ctx, const amoe_group* grp, void* stream);

/* a8 (+a1/a2 of the next layer): drain this rank's combine ring; per token h += Σ_k w_k O_k
 * (+ shared outputs), fixed ascending order, fp32 multiply/add without FMA, stored; x =
 * rmsnorm(h); layer+1 (after the last layer: pass+1, layer 0); retire when pass == retire_pass
 * else route with the router table and enqueue. */
amoe_status amoe_combine(amoe_ctx_t ctx, int retire_pass, void* stream);

/* Run the asynchronous scheduler loop (host C++; "whenever the GPU becomes idle",
 * Algorithm 1) until every token of every rank has retired at pass `retire_pass`:
 * read the queue counters, pick (params->policy: Algorithm 1 with lookahead W and δ, MTFS,
 * FLFS, the lockstep SYNC baseline, or Algorithm 1 with the box-wide lookahead), execute, merge.
 * A pick is one (layer, expert) queue, or with params->grouped every nonempty hosted queue of
 * the picked layer. Execution: a cold pick (every queue <= 16 legs, <= 32 for Mixtral-sized
 * experts or groups of >= 4; bf16, d % 256 == 0) runs amoe_execute_cold, otherwise
 * amoe_rebatch_ffn_forward; then amoe_combine. Asynchronous policies pipeline the loop: the host
 * decides pick k + 1 from an asynchronous counter snapshot while pick k runs (every drain takes
 * exactly the host's count); AMOE_PIPELINE=0 synchronises after each pick.
 * params->max_picks > 0 (single rank, not SYNC): return after that many picks or when nothing is
 * runnable (open-loop stepping; the caller admits new tokens between calls).
 * Returns AMOE_OK; AMOE_EINVAL for bad params, a missing router (neither table nor gate), a
 * hosted queue without weights, SYNC with stepping, stepping at G > 1; AMOE_EPEER before
 * amoe_import_peers at G > 1; AMOE_EDEVICE when a device fault is latched (amoe_error_info):
 * any kernel fault, a lost leg at G = 1 (code 11, naming the stranded token), a peer's fault at
 * G > 1 (code 9: the faulting rank stores an abort mark into every peer, so every rank returns),
 * or AMOE_RUN_TIMEOUT seconds (default 600) without completion at G > 1 (code 10). Multi-GPU:
 * keeps serving peers until all ranks report done. stats may be NULL. */
amoe_status amoe_run(amoe_ctx_t ctx, const amoe_run_params* params, int retire_pass,
                     amoe_run_stats* stats, void* stream);

/* One decode pass end-to-end from HOST buffers: h0_host [T_slots, d] storage dtype (all slots)
 * is copied in, and router_host [L][T_slots][E] fp32 (or NULL to keep the resident table) is
 * copied into router table (pass mod n_tables; layer 0 routes with its gate instead when
 * amoe_set_gate gave it one); every token runs layers 0..L-1 once
 * (amoe_token_init + amoe_enqueue(layer 0) + amoe_run) and the final h is copied to
 * h_out_host [T_slots, d]. Synchronises `stream`. Multi-GPU: every rank calls it. */
amoe_status amoe_pass_host(amoe_ctx_t ctx, const void* h0_host, const float* router_host, void* h_out_host,
                           int pass, const amoe_run_params* params, amoe_run_stats* stats, void* stream);

/* Per-stage device timing: when enabled, CUDA events bracket every launch of each stage on its
 * stream (no synchronisation added). enable resets the accumulators (synchronises the device).
 * read synchronises on the recorded events and returns summed milliseconds and the number of
 * timed launches per stage: [0] rebatch (drain+gather), [1] FFN gate/up+SwiGLU, [2] FFN down,
 * [3] forward, [4] combine (+route/scatter), [5] token_init/enqueue, [6..7] reserved. */
amoe_status amoe_profile_enable(amoe_ctx_t ctx, int enable);
amoe_status amoe_profile_read(amoe_ctx_t ctx, double ms_out[8], int64_t counts_out[8]);
/* Expert executions amoe_run performed while profiling was enabled (reset by
 * amoe_profile_enable): pairs out[2i] = layer * H + local queue, out[2i+1] = legs drained by that
 * execution (taken from consecutive ring-head snapshots, so exact). Copies min(cap, *n_out)
 * pairs; *n_out = executions logged. For the schedule-conditional roofline. */
amoe_status amoe_exec_log(amoe_ctx_t ctx, int32_t* out, int cap, int* n_out);

/* ---- introspection -------------------------------------------------------------------- */

typedef enum amoe_buffer_id {
  AMOE_BUF_H = 0,         /* [T_slots, d] residual stream h */
  AMOE_BUF_X = 1,         /* [T_slots, d] rmsnorm(h): what experts read */
  AMOE_BUF_POOL = 2,      /* [T_slots, K+S, d] returned legs */
  AMOE_BUF_TOK_W = 3,     /* [T_slots, K] fp32 routing weights of the current layer */
  AMOE_BUF_TOK_IDX = 4,   /* [T_slots, K] int32 routed experts of the current layer */
  AMOE_BUF_TOK_LAYER = 5, /* [T_slots] int32 current layer */
  AMOE_BUF_TOK_PASS = 6,  /* [T_slots] int32 current pass */
  AMOE_BUF_RINGS = 7,     /* [L*H][ring_cap] amoe_leg */
  AMOE_BUF_QCTR = 8,      /* [L*H][4] uint32 {reserve, commit, head, pad} */
  AMOE_BUF_STATS = 9,     /* uint64 [8]: merges, retired, legs_forwarded, ... */
  AMOE_BUF_SCRATCH = 10,  /* the internal amoe_group buffers used by amoe_run (tile first) */
  AMOE_BUF_TOK_TIME = 11  /* [T_slots][2] uint64 device globaltimer ns: admission (amoe_token_init)
                             and retirement (the combine that retires the token): per-token latency */
} amoe_buffer_id;

amoe_status amoe_get_buffer(amoe_ctx_t ctx, int which, void** dev_ptr, size_t* bytes);
int amoe_hosted(amoe_ctx_t ctx);        /* H = queues per layer per rank (routed max + S) */
int amoe_ring_cap(amoe_ctx_t ctx);      /* entries per µ-queue ring */
/* local queue index of (layer-independent) expert e on its owner; -1 if invalid. */
int amoe_local_queue(amoe_ctx_t ctx, int expert);
/* fill the internal group scratch (amoe_run's buffers) into *grp, nq = 0. */
amoe_status amoe_scratch_group(amoe_ctx_t ctx, amoe_group* grp);
/* number of libamoe kernel launches issued by this context so far. */
int64_t amoe_launch_count(amoe_ctx_t ctx);

/* SMs per die of the current device as measured by the library's L2-latency probe (run once per
 * device at the first amoe_create): counts[1] == 0 means no die split was detected. The split
 * is used by the optional die-aware FFN schedule (AMOE_FFN_SCHED=die); the
 * default dynamic schedule does not need it. AMOE_DIE_PROBE=0 skips the probe. */
amoe_status amoe_die_info(int32_t counts[2]);

/* Synchronise the context's last stream and report a latched device fault (AMOE_EDEVICE). */
amoe_status amoe_check(amoe_ctx_t ctx);
/* info[0] = fault code, info[1..3] = fault arguments. */
amoe_status amoe_error_info(amoe_ctx_t ctx, uint32_t info[4]);
/* Clear the latched fault (tests). */
amoe_status amoe_clear_error(amoe_ctx_t ctx);
const char* amoe_status_string(amoe_status s);
/* Teardown; frees host-side state only (never caller memory). */
amoe_status amoe_destroy(amoe_ctx_t ctx);

#ifdef __cplusplus
}
#endif
#endif /* AMOE_H */
