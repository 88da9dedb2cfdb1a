// k_ffn_cold.cu — a4 + a5 + a6 + a7 fused for COLD picks (every queue of the pick holds <= 128
// tokens): one persistent launch drains the queues, gathers the tokens' x rows, runs the SwiGLU
// expert (gate/up, SwiGLU, down) and stores each output row straight into its home's token pool
// (one-sided, NVLink peer store when remote), counting the leg's columns for the merge.
//
// Why a separate kernel (small batches make expert execution weight-loading
// bound): with <= 128 tokens per expert the work is streaming the expert's
// weights (6·d·ff bytes) from HBM once, and four launches (drain, gather, gate/up, down) with
// their prologues, tails and split-K reductions cost more than the streaming itself (one
// DeepSeek expert: 17 MB = 2.6 us at HBM speed). Design, B200-first:
//  * swap-AB tcgen05 MMA: the weight tile is the M = 128 operand and the tokens are N = n_pad
//    (16..128), so a cold expert does not pay a 128/256-row token tile;
//  * gate/up: two MMAs per K step (W1 and W3 slabs against the same token tile) into two TMEM
//    accumulators, SwiGLU in registers; down: two K blocks per stage so every stage streams the
//    same 32 KB of weights;
//  * stream-K over weight bytes: CTA c of P takes iterations [c·I/P, (c+1)·I/P) of each phase
//    (I = gate/up K-block slabs, then down slabs), so all SMs stream equal bytes whatever the
//    number of experts and tiles; a tile split across CTAs is reduced in parallel (each of its
//    nseg owners sums 1/nseg of its rows over all owners' fp32 partials in a fixed order:
//    deterministic) — no cross-CTA atomics on values;
//  * the producer streams the first stages' weights BEFORE the grid dependency wait (weights
//    are constant), overlapping the previous kernel's tail and the drain/gather latency;
//  * dependencies inside the launch are per tile: a down slab waits only for the act columns
//    it reads (a counter per gate/up tile), the token tile for the grid-wide gather.
// All CTAs are co-resident (one per SM, grid <= SMs), every wait is on work that cannot itself
// wait on the waiter, so the in-kernel dependencies cannot deadlock.
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "amoe_internal.cuh"
#include "tc_ptx.cuh"

namespace amoe {
namespace cold {
using namespace tc;

constexpr int THREADS = 256;
constexpr int MAXS = 8;               // smem ring stages (runtime count)
constexpr int NMAX = 128;             // tokens per queue (MMA N, padded to 16)
constexpr int A_BYTES = 128 * 64 * 2; // one 128-row x 64-col bf16 weight box (16 KB)
constexpr int MAXP = 256;             // CTAs (flags are indexed by CTA)
constexpr int SMEM_DYN = 216 * 1024;  // dynamic smem request (ring + 1 KB alignment slack)
constexpr int RING_BUDGET = SMEM_DYN - 1024;
// counters (u32, workspace `cold`): [0] drain flag, [1] gather arrivals, [2] exits,
// [16 + (phase*2 + which)*MAXP + cta] partial-ready tags, [kActQ + q] act tokens·tiles done
constexpr int kPartFlag = 16;
constexpr int kActQ = kPartFlag + 4 * MAXP;
constexpr int kPartFloats = NMAX * 256;   // one partial slot: [token][256] fp32 (128 KB)

struct ColdArgs {
  int32_t nq, n_pad, stages;
  int32_t ipt_a, ipt_b;       // iterations per tile: d/64 (gate/up), ff/128 (down, 2 K blocks each)
  int32_t ft, dt;             // tiles per queue: ff/128 (gate/up), d/128 (down)
  int32_t ia, ib;             // iterations per phase (all queues)
  int32_t pa, pb;             // CTAs streaming each phase (<= grid)
  int32_t sa, sb;             // units per tile of each phase (1 = whole tiles)
  uint32_t seq;               // launch tag for the partial-ready flags
  uint32_t* ctr;              // workspace counters (see above)
  float* part;                // partial slots [(phase*2 + which)*MAXP + cta][kPartFloats]
  int32_t* qinfo;             // [3*AMOE_MAX_GROUP]: drained n, row offset, ring start per queue
  __nv_bfloat16* tile;        // [nq*n_pad][d]: gathered token rows
  __nv_bfloat16* act;         // [nq*n_pad][ff]: SwiGLU activations
  const CUtensorMap* wmaps;   // [L*H][3]
  int32_t qid[AMOE_MAX_GROUP];   // l*H + lq
  int32_t cap[AMOE_MAX_GROUP];   // drain at most this many legs (the scheduler's snapshot)
};

// Partition of one phase's iterations (tiles x ipt) over its P CTAs: with
// tiles <= SMs every tile is cut into s = P / tiles contiguous units, one per CTA; with more
// tiles than SMs each CTA takes a contiguous run of whole tiles. A CTA's range starts at unit
// floor(c·U/P) (U = tiles·s); unit u starts at iteration (u / s)·ipt + floor((u mod s)·ipt / s).
struct Part {
  int tiles, ipt, s, P;
  __device__ __forceinline__ int start(int c) const {
    const int u = (int)((int64_t)c * (tiles * s) / P);
    const int t = u / s, r = u - t * s;
    return t * ipt + (r * ipt) / s;
  }
  // CTA whose range holds iteration it (the largest c with start(c) <= it)
  __device__ __forceinline__ int owner(int it) const {
    if (s == ipt) {   // one iteration per unit (stream-K): closed form
      const int I = tiles * ipt;
      const int c = (int)(((int64_t)(it + 1) * P - 1) / I);
      return c < P - 1 ? c : P - 1;
    }
    int lo = 0, hi = P - 1;
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (start(mid) <= it) lo = mid; else hi = mid - 1; }
    return lo;
  }
};

__device__ __forceinline__ uint32_t ld_acq_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_rel_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// In-kernel waits are bounded: a wait that has not been satisfied after kWatchdogNs is a bug
// (a dependency that can never complete); the kernel traps instead of hanging the GPU, so the
// launch fails with an error the host sees (cudaErrorLaunchFailure -> AMOE_ECUDA).
constexpr uint64_t kWatchdogNs = 4000000000ull;
__device__ __noinline__ void watchdog_trap(uint32_t where) {
  printf("amoe cold kernel watchdog: block %d thread %d wait %u\n", blockIdx.x, threadIdx.x, where);
  asm volatile("trap;");
}
__device__ __forceinline__ uint32_t ld_rlx_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Poll with relaxed loads (no sleep: every wait here is on the critical path of the launch),
// then one fence orders everything after the observation (acquire pattern).
__device__ __forceinline__ void spin_until_eq(const uint32_t* p, uint32_t v, uint32_t where = 0) {
  if (ld_rlx_gpu(p) != v) {
    const uint64_t t0 = globaltimer_ns();
    for (uint32_t i = 1;; ++i) {
      if (ld_rlx_gpu(p) == v) break;
      if ((i & 1023u) == 0 && globaltimer_ns() - t0 > kWatchdogNs) watchdog_trap(where);
    }
  }
  fence_acq_gpu();
}
// The TMA producer observes dependencies with acquire LOADS, never a fence: a fence would wait
// for the thread's outstanding bulk copies and drain the weight pipeline.
__device__ __forceinline__ bool test_eq_acq(const uint32_t* p, uint32_t v) { return ld_acq_gpu(p) == v; }
__device__ __forceinline__ void spin_until_eq_acq(const uint32_t* p, uint32_t v, uint32_t where) {
  if (ld_acq_gpu(p) == v) return;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t i = 1;; ++i) {
    if (ld_acq_gpu(p) == v) return;
    if ((i & 1023u) == 0 && globaltimer_ns() - t0 > kWatchdogNs) watchdog_trap(where);
  }
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
               : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_wd(uint32_t bar, uint32_t parity, uint32_t where) {
  uint32_t ok;
  asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\nselp.u32 %0, 1, 0, P1;\n}\n"
               : "=r"(ok) : "r"(bar), "r"(parity), "r"(kSuspendNs) : "memory");
  if (ok) return;
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\nselp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(ok) : "r"(bar), "r"(parity), "r"(kSuspendNs) : "memory");
    if (ok) return;
    if (globaltimer_ns() - t0 > kWatchdogNs) watchdog_trap(where);
  }
}
// generic-proxy stores (act, gathered rows) -> visible to TMA (async proxy) reads elsewhere
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }   // warps 4..7
__device__ __forceinline__ void gat_bar() { asm volatile("bar.sync 2, 192;" ::: "memory"); }   // warps 2..7

// The CTA's j-th item (phase A items first, then phase B).
struct Items {
  int a0, a1, b0, b1, ipt_a, ipt_b;
  __device__ __forceinline__ int count() const { return (a1 - a0) + (b1 - b0); }
  __device__ __forceinline__ void get(int j, int& phase, int& tile, int& k) const {
    if (j < a1 - a0) { const int it = a0 + j; phase = 0; tile = it / ipt_a; k = it - tile * ipt_a; }
    else { const int it = b0 + j - (a1 - a0); phase = 1; tile = it / ipt_b; k = it - tile * ipt_b; }
  }
  // first / last item of its segment
  __device__ __forceinline__ bool seg_first(int j) const {
    int ph, t, k;
    get(j, ph, t, k);
    return k == 0 || j == 0 || j == a1 - a0;
  }
  __device__ __forceinline__ bool seg_last(int j) const {
    int ph, t, k;
    get(j, ph, t, k);
    const int ipt = ph == 0 ? ipt_a : ipt_b;
    return k == ipt - 1 || j == count() - 1 || j == a1 - a0 - 1;
  }
};

// (which) slot of CTA o's segment in tile t: 0 when o's range starts inside t (its first
// segment of the phase, k0 > 0), else 1 (its last segment, k0 == 0)
__device__ __forceinline__ int which_of(int o, int t, const Part& pt) { return pt.start(o) > t * pt.ipt ? 0 : 1; }

#ifdef AMOE_COLD_TRACE
// diagnostic build only: per-CTA globaltimer stamps of the last launch (tools/cold_trace.py)
__device__ unsigned long long g_cold_trace[16][MAXP];
#define CT(i) (g_cold_trace[i][blockIdx.x] = globaltimer_ns())
#else
#define CT(i) ((void)0)
#endif

__global__ void __launch_bounds__(THREADS, 1)
ffn_cold_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmAct,
                const __grid_constant__ ColdArgs a, const __grid_constant__ DevCtx dc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (threadIdx.x == 0) CT(0);
  __shared__ uint64_t bars[2 * MAXS + 4];      // full[MAXS], empty[MAXS], tfull[2], tempty[2]
  __shared__ uint32_t tmem_holder[4];
  __shared__ int s_n[AMOE_MAX_GROUP], s_start[AMOE_MAX_GROUP];
  __shared__ int s_pend[2][4][4];              // per phase: up to 2 split segments {tile, k0, k1, -}
  __shared__ int s_npend[2];
  __shared__ unsigned long long s_dst[NMAX];   // pool row of each token of s_dstq (down epilogue)
  __shared__ __align__(16) __nv_bfloat16 s_stage[16][128];   // epilogue transpose (16 tokens)
  __shared__ int s_dstq;
  __shared__ int s_last;
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = gridDim.x, cta = blockIdx.x;
  const int n_pad = a.n_pad, S = a.stages;
  const int stage_bytes = 2 * A_BYTES + 2 * n_pad * 128;
  // phase X is streamed by CTAs [0, P_X): CTA c takes iterations [c·I/P_X, (c+1)·I/P_X)
  const Part part_a{a.ia / a.ipt_a, a.ipt_a, a.sa, a.pa}, part_b{a.ib / a.ipt_b, a.ipt_b, a.sb, a.pb};
  const bool in_a = cta < a.pa, in_b = cta < a.pb;
  const Items it{in_a ? part_a.start(cta) : 0, in_a ? part_a.start(cta + 1) : 0, in_b ? part_b.start(cta) : 0,
                 in_b ? part_b.start(cta + 1) : 0, a.ipt_a, a.ipt_b};
  const int n_items = it.count();
  uint32_t* ctr = a.ctr;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(smem_u32(&bars[s]), 1); mbar_init(smem_u32(&bars[MAXS + s]), 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(smem_u32(&bars[2 * MAXS + b]), 1); mbar_init(smem_u32(&bars[2 * MAXS + 2 + b]), 1); }
    s_npend[0] = s_npend[1] = 0;
    s_dstq = -1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_holder)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem_base = tmem_holder[0];
  const uint32_t idesc = idesc_bf16(128, n_pad);

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer
      // A (weights) of an item, and its B (tokens / activations) once its dependency holds
      const uint64_t wpol = policy_evict_first();
      auto issue_a = [&](int j, int s) {
        int ph, t, k;
        it.get(j, ph, t, k);
        const uint32_t sa = smem_u32(ring + s * stage_bytes);
        const uint32_t full = smem_u32(&bars[s]);
        mbar_expect_tx(full, 2 * A_BYTES + (ph == 0 ? 1 : 2) * n_pad * 128);
        if (ph == 0) {
          const int q = t / a.ft, f = t - q * a.ft;
          const CUtensorMap* wm = a.wmaps + a.qid[q] * 3;
          tma_load_2d_hint(sa, wm, k * 64, f * 128, full, wpol);
          tma_load_2d_hint(sa + A_BYTES, wm + 1, k * 64, f * 128, full, wpol);
        } else {
          const int q = t / a.dt, dtl = t - q * a.dt;
          const CUtensorMap* wm = a.wmaps + a.qid[q] * 3 + 2;
          tma_load_2d_hint(sa, wm, (2 * k) * 64, dtl * 128, full, wpol);
          tma_load_2d_hint(sa + A_BYTES, wm, (2 * k + 1) * 64, dtl * 128, full, wpol);
        }
      };
      bool gathered = false;
      int ready_q = -1;                               // queue whose activations are all stored
      // dependency of an item's B operand: the token tile (phase A: the grid-wide gather) or the
      // queue's activations (phase B: every gate/up tile of the queue finalised for its n tokens,
      // counted in tokens x tiles); observed once, then one proxy fence orders the TMA reads
      auto dep_ok = [&](int j, bool block) -> bool {
        int ph, t, k;
        it.get(j, ph, t, k);
        if (ph == 0) {
          if (!gathered) {
            if (block) spin_until_eq_acq(ctr + 1, (uint32_t)P, 5);
            else if (!test_eq_acq(ctr + 1, (uint32_t)P)) return false;
            proxy_fence();
            gathered = true;
          }
          return true;
        }
        const int q = t / a.dt;
        if (q == ready_q) return true;
        const uint32_t need = (uint32_t)(a.ft * ld_acq_gpu(reinterpret_cast<const uint32_t*>(a.qinfo) + q));
        if (block) spin_until_eq_acq(ctr + kActQ + q, need, 6);
        else if (!test_eq_acq(ctr + kActQ + q, need)) return false;
        proxy_fence();
        ready_q = q;
        return true;
      };
      auto issue_b = [&](int j, int s) {
        int ph, t, k;
        it.get(j, ph, t, k);
        const uint32_t sb = smem_u32(ring + s * stage_bytes) + 2 * A_BYTES;
        const uint32_t full = smem_u32(&bars[s]);
        if (ph == 0) {
          const int q = t / a.ft;
          tma_load_2d(sb, &tmX, k * 64, q * n_pad, full);
        } else {
          const int q = t / a.dt;
          tma_load_2d(sb, &tmAct, (2 * k) * 64, q * n_pad, full);
          tma_load_2d(sb + n_pad * 128, &tmAct, (2 * k + 1) * 64, q * n_pad, full);
        }
      };
      // weights of the first stages stream before the grid dependency (they are constant)
      int pend[MAXS], ps[MAXS], np = 0, ph0 = 0;
      int stage = 0;
      uint32_t phase = 0;
      int j = 0;
      for (; j < n_items && j < S; ++j) {
        issue_a(j, stage);
        pend[(ph0 + np) % MAXS] = j; ps[(ph0 + np) % MAXS] = stage; ++np;
        if (++stage == S) { stage = 0; phase ^= 1u; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      CT(1);
      bool b_first = true, bb_first = true;
      for (;;) {
        // B loads of pending items, in order, as their dependencies hold: polled without blocking
        // while a free stage can take the next item's weights, blocking once every stage waits
        // for its B (the MMA consumes the stages in order) or nothing is left to prefetch
        if (np > 0) {
          bool stuck = np == S || j >= n_items || !mbar_test(smem_u32(&bars[MAXS + stage]), phase ^ 1u);
          while (np > 0 && dep_ok(pend[ph0], stuck)) {
            {
              int ph_, t_, k_;
              it.get(pend[ph0], ph_, t_, k_);
              if (ph_ == 0 && b_first) { CT(4); b_first = false; }
              if (ph_ == 1 && bb_first) { CT(8); bb_first = false; }
            }
            issue_b(pend[ph0], ps[ph0]);
            ph0 = (ph0 + 1) % MAXS; --np;
          }
        }
        if (j >= n_items) {
          if (np == 0) break;
          continue;
        }
        mbar_wait_wd(smem_u32(&bars[MAXS + stage]), phase ^ 1u, 1);
        issue_a(j, stage);
        pend[(ph0 + np) % MAXS] = j; ps[(ph0 + np) % MAXS] = stage; ++np;
        ++j;
        if (++stage == S) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0) {
      // ===================== MMA issuer (single thread): swap-AB, D[128 weight rows][n_pad tokens]
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int j = 0; j < n_items; ++j) {
        int ph, t, k;
        it.get(j, ph, t, k);
        const bool first = it.seg_first(j), last = it.seg_last(j);
        if (first) {
          mbar_wait_wd(smem_u32(&bars[2 * MAXS + 2 + acc]), acc_phase ^ 1u, 2);
          tc_fence_after();
        }
        const uint32_t d0 = tmem_base + (uint32_t)(acc * 256);
        mbar_wait_wd(smem_u32(&bars[stage]), phase, 3);
        tc_fence_after();
        const uint32_t sa = smem_u32(ring + stage * stage_bytes);
        const uint64_t a0d = umma_desc_sw128(sa), a1d = umma_desc_sw128(sa + A_BYTES);
        const uint64_t b0d = umma_desc_sw128(sa + 2 * A_BYTES), b1d = umma_desc_sw128(sa + 2 * A_BYTES + n_pad * 128);
        if (ph == 0) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t accum = (!first || kk > 0) ? 1u : 0u;
            umma_bf16(d0, a0d + 2 * kk, b0d + 2 * kk, idesc, accum);              // gate
            umma_bf16(d0 + (uint32_t)n_pad, a1d + 2 * kk, b0d + 2 * kk, idesc, accum);   // up
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16(d0, a0d + 2 * kk, b0d + 2 * kk, idesc, (!first || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16(d0, a1d + 2 * kk, b1d + 2 * kk, idesc, 1u);
        }
        umma_commit(smem_u32(&bars[MAXS + stage]));
        if (++stage == S) { stage = 0; phase ^= 1u; }
        if (last && j == it.a1 - it.a0 - 1) CT(5);
        if (last) {
          umma_commit(smem_u32(&bars[2 * MAXS + acc]));
          if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        }
      }
      CT(9);
    }
  } else {
    // ===================== warps 2..7: drain (CTA 0, warp 3), gather, then (4..7) epilogue
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (cta == 0 && warp == 3) {
      uint32_t tot = 0;
      for (int q = lane; q < a.nq; q += 32) {
        uint32_t* qc = qctr_ptr(dc, dc.rank, a.qid[q]);
        const uint32_t cm = ld_acquire(qc + 1);
        const uint32_t rv = ld_relaxed(qc + 0);
        const uint32_t head = qc[2];
        if (rv - head > dc.ring_cap) raise_fault(dc, F_RING_OVERFLOW, a.qid[q], rv, head);
        uint32_t n;
        const uint32_t cap = (uint32_t)a.cap[q];
        if (cm == rv) {
          n = cm - head;
        } else {   // a producer on a peer is mid-flight: the published prefix is where seq == pos + 1
          const amoe_leg* rg = ring_ptr(dc, dc.rank, a.qid[q]);
          n = 0;
          while (n < cap && n < rv - head && ld_acquire(&rg[(head + n) & dc.ring_mask].seq) == head + n + 1u) ++n;
        }
        if (n > cap) n = cap;
        a.qinfo[q] = (int32_t)n;                                  // amoe_group qinfo layout:
        a.qinfo[AMOE_MAX_GROUP + q] = q * n_pad;                  // n, row offset, ring start
        a.qinfo[2 * AMOE_MAX_GROUP + q] = (int32_t)head;
        qc[2] = head + n;
        tot += n;
      }
      __syncwarp();
      if (dc.xlog) {
        // checked mode: one record per nonempty queue + its legs (seq := the token's pass)
        uint32_t* xl = dc.xlog;
        for (int q = 0; q < a.nq; ++q) {
          const uint32_t n = (uint32_t)a.qinfo[q], head = (uint32_t)a.qinfo[2 * AMOE_MAX_GROUP + q];
          if (!n) continue;
          uint32_t e0 = 0, l0 = 0;
          if (lane == 0) {
            e0 = atomicAdd(xl + 0, 1u);
            l0 = atomicAdd(xl + 1, n);
            if (e0 < xl[2]) {
              uint32_t* r = xlog_exec(xl) + 4 * (uint64_t)e0;
              r[0] = (uint32_t)a.qid[q]; r[1] = head; r[2] = n; r[3] = l0;
            }
          }
          l0 = __shfl_sync(0xffffffffu, l0, 0);
          const amoe_leg* rg = ring_ptr(dc, dc.rank, a.qid[q]);
          for (uint32_t i = lane; i < n; i += 32) {
            if (l0 + i >= xl[3]) break;
            amoe_leg e = rg[(head + i) & dc.ring_mask];
            const int home = (e.home >= 0 && e.home < dc.G) ? e.home : dc.rank;
            const int slot = (e.token_slot >= 0 && e.token_slot < dc.T) ? e.token_slot : 0;
            e.seq = (uint32_t)reinterpret_cast<const int32_t*>(dc.peer[home] + dc.lay.tok_pass)[slot];
            xlog_legs(xl)[l0 + i] = e;
          }
          __syncwarp();
        }
      }
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (lane == 0) {
        atomicAdd(wsp<unsigned long long>(dc, dc.rank, dc.lay.stats) + 2, (unsigned long long)tot);
        __threadfence();
        st_rel_gpu(ctr + 0, 1u);
      }
    }
    if (lane == 0) spin_until_eq(ctr + 0, 1u, 7);
    __syncwarp();
    if (warp == 2 && lane == 0) CT(2);
    if (warp == 2)
      for (int q = lane; q < a.nq; q += 32) { s_n[q] = a.qinfo[q]; s_start[q] = a.qinfo[2 * AMOE_MAX_GROUP + q]; }
    gat_bar();
    // gather: warp-per-row copy of each drained leg's x row (local, or from its home over
    // NVLink) into the contiguous token tile, row q*n_pad + i
    {
      const int rowbytes = dc.d * 2;
      const int gw = cta * 6 + (warp - 2), nw = P * 6;
      uint32_t remote = 0;
      for (int r = gw; r < a.nq * n_pad; r += nw) {
        const int q = r / n_pad, i = r - q * n_pad;
        if (i >= s_n[q]) continue;
        const uint32_t pos = (uint32_t)s_start[q] + (uint32_t)i;
        const amoe_leg e = ring_ptr(dc, dc.rank, a.qid[q])[pos & dc.ring_mask];
        if (e.seq != pos + 1u || e.home < 0 || e.home >= dc.G || e.token_slot < 0 || e.token_slot >= dc.T) {
          if (lane == 0) raise_fault(dc, F_STALE_ENTRY, a.qid[q], pos, e.seq);
          continue;
        }
        remote += (e.home != dc.rank);
        warp_copy(a.tile + (uint64_t)r * dc.d,
                  reinterpret_cast<const char*>(dc.peer[e.home] + dc.lay.x) + (uint64_t)e.token_slot * rowbytes,
                  rowbytes, lane);
      }
      proxy_fence();
      __threadfence();
      if (lane == 0 && remote)
        atomicAdd(wsp<unsigned long long>(dc, dc.rank, dc.lay.stats) + 3, (unsigned long long)remote);
      gat_bar();
      if (warp == 2 && lane == 0) { red_rel_gpu(ctr + 1, 1u); CT(3); }
    }
    if (warp >= 4) {
      // ===================== epilogue (warps 4..7): TMEM lane quarter ew, weight row r
      const int ew = warp - 4, r = ew * 32 + lane, et = tid - 128;
      const bool sys = dc.G > 1;
      int acc = 0;
      uint32_t acc_phase = 0;
      // pool row of every token of queue q (down epilogue destinations), cached in smem
      auto load_dst = [&](int q) {
        if (s_dstq == q) return;
        epi_bar();
        if (et < s_n[q]) {
          const amoe_leg e = ring_ptr(dc, dc.rank, a.qid[q])[((uint32_t)s_start[q] + (uint32_t)et) & dc.ring_mask];
          s_dst[et] = dc.peer[e.home] + dc.lay.pool + ((uint64_t)e.token_slot * dc.KS + (uint64_t)e.k) * dc.d * 2;
        }
        epi_bar();
        if (et == 0) s_dstq = q;
        epi_bar();
      };
      auto count_cols = [&](int q, int t, uint32_t cols) {
        const amoe_leg e = ring_ptr(dc, dc.rank, a.qid[q])[((uint32_t)s_start[q] + (uint32_t)t) & dc.ring_mask];
        leg_pieces_done(dc, e.home, e.token_slot, e.k, cols);
      };
      int j = 0;
      for (int phz = 0; phz < 2; ++phz) {
        const int jend = phz == 0 ? (it.a1 - it.a0) : n_items;
        const int ipt = phz == 0 ? a.ipt_a : a.ipt_b;
        const Part& pt = phz == 0 ? part_a : part_b;
        // ---- segments of this phase
        while (j < jend) {
          int ph, t, k0;
          it.get(j, ph, t, k0);
          int jl = j;
          while (!it.seg_last(jl)) ++jl;
          int ph1, t1, kl;
          it.get(jl, ph1, t1, kl);
          const int k1 = kl + 1;
          j = jl + 1;
          const uint32_t tfull = smem_u32(&bars[2 * MAXS + acc]);
          const uint32_t tempty = smem_u32(&bars[2 * MAXS + 2 + acc]);
          if (et == 0) {
            mbar_wait_wd(tfull, acc_phase, 4);
            if (ph == 0 && j == jend) CT(12);
          }
          epi_bar();
          tc_fence_after();
          const uint32_t tb = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(ew * 32) << 16);
          const int q = ph == 0 ? t / a.ft : t / a.dt;
          const int tl = ph == 0 ? t - q * a.ft : t - q * a.dt;
          const int n = s_n[q];
          const bool whole = k0 == 0 && k1 == ipt;
          if (ph == 1 && whole) load_dst(q);
          const int which = k0 > 0 ? 0 : 1;
          float* part = a.part + (size_t)((ph * 2 + which) * MAXP + cta) * kPartFloats;
          for (int c0 = 0; c0 < n; c0 += 16) {
            float v[32];
            if (ph == 0) tmem_ld16x2(tb + c0, tb + n_pad + c0, v);     // v[0..16) gate, v[16..32) up
            else tmem_ld16(tb + c0, v);
            const int m = min(16, n - c0);
            if (whole) {
              // thread r holds column r of 16 token rows: transpose through smem, then every row
              // (256 B: the tile's 128 columns) leaves as 16-B vector stores
              for (int i = 0; i < m; ++i)
                s_stage[i][r] = __float2bfloat16_rn(ph == 0 ? silu_mul(v[i], v[16 + i]) : v[i]);
              epi_bar();
              for (int x = et; x < m * 16; x += 128) {
                const int tk = x >> 4, cc = x & 15;
                const uint4 val = reinterpret_cast<const uint4*>(s_stage[tk])[cc];
                __nv_bfloat16* dst = ph == 0 ? a.act + (uint64_t)(q * n_pad + c0 + tk) * dc.ff + tl * 128
                                             : reinterpret_cast<__nv_bfloat16*>(s_dst[c0 + tk]) + tl * 128;
                reinterpret_cast<uint4*>(dst)[cc] = val;
              }
              epi_bar();
            } else {
              for (int i = 0; i < m; ++i) {
                float* row = part + (size_t)(c0 + i) * 256;
                row[r] = v[i];
                if (ph == 0) row[128 + r] = v[16 + i];
              }
            }
          }
          tc_fence_before();
          epi_bar();
          if (et == 0) mbar_arrive(tempty);        // TMEM buffer free for the MMA
          if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
          // publish: act tile / leg columns / partial
          if (ph == 0 || !whole) proxy_fence();
          if (whole && ph == 1) fence_sc(sys); else __threadfence();
          epi_bar();
          if (whole) {
            if (ph == 0) { if (et == 0 && n > 0) red_rel_gpu(ctr + kActQ + q, (uint32_t)n); }
            else if (et < n) count_cols(q, et, 128u);
          } else {
            if (et == 0) {
              st_rel_gpu(ctr + kPartFlag + (ph * 2 + which) * MAXP + cta, a.seq);
              const int np = s_npend[ph];
              s_pend[ph][np][0] = t; s_pend[ph][np][1] = k0; s_pend[ph][np][2] = k1;
              s_npend[ph] = np + 1;
            }
            epi_bar();
          }
        }
        if (et == 0) { if (phz == 0) CT(6); }
        // ---- reductions of this phase's split tiles: owner j of the tile's nseg owners sums, for
        // tokens [j·n/nseg, (j+1)·n/nseg), every row over all owners' fp32 partials in owner
        // order (deterministic), float4 at a time with the owners' loads in flight together
        epi_bar();
        const int npend = s_npend[phz];
        for (int pi = 0; pi < npend; ++pi) {
          const int t = s_pend[phz][pi][0];
          const int first = pt.owner(t * ipt), last = pt.owner(t * ipt + ipt - 1);
          const int nseg = last - first + 1, jj = cta - first;
          const int q = phz == 0 ? t / a.ft : t / a.dt;
          const int tl = phz == 0 ? t - q * a.ft : t - q * a.dt;
          const int n = s_n[q];
          const int t0 = jj * n / nseg, t1 = (jj + 1) * n / nseg;
          if (et < nseg) {
            const int o = first + et;
            spin_until_eq(ctr + kPartFlag + (phz * 2 + which_of(o, t, pt)) * MAXP + o, a.seq, 8);
          }
          epi_bar();
          if (et == 0 && pi == 0 && phz == 0) CT(13);
          if (et == 0 && pi == 0 && phz == 1) CT(14);
          if (phz == 1) load_dst(q);
          const int items = (t1 - t0) * 32;                // (token, 4-row chunk)
          for (int x0 = et; x0 < items; x0 += 128 * 2) {
            float4 g[2], u[2];
            int tok[2], ch[2];
            bool ok[2];
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int x = x0 + v * 128;
              ok[v] = x < items;
              tok[v] = t0 + (x >> 5); ch[v] = x & 31;
              g[v] = make_float4(0.f, 0.f, 0.f, 0.f); u[v] = g[v];
            }
            for (int ob = first; ob <= last; ob += 4) {
              float4 pg[4][2], pu[4][2];
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                  if (ob + i <= last && ok[v]) {
                    const float* row = a.part +
                                       (size_t)((phz * 2 + which_of(ob + i, t, pt)) * MAXP + ob + i) * kPartFloats +
                                       (size_t)tok[v] * 256 + 4 * ch[v];
                    pg[i][v] = *reinterpret_cast<const float4*>(row);
                    if (phz == 0) pu[i][v] = *reinterpret_cast<const float4*>(row + 128);
                  }
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                  if (ob + i <= last && ok[v]) {
                    g[v].x += pg[i][v].x; g[v].y += pg[i][v].y; g[v].z += pg[i][v].z; g[v].w += pg[i][v].w;
                    if (phz == 0) { u[v].x += pu[i][v].x; u[v].y += pu[i][v].y; u[v].z += pu[i][v].z; u[v].w += pu[i][v].w; }
                  }
            }
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              if (!ok[v]) continue;
              __nv_bfloat162 o2[2];
              if (phz == 0) {
                o2[0] = __floats2bfloat162_rn(silu_mul(g[v].x, u[v].x), silu_mul(g[v].y, u[v].y));
                o2[1] = __floats2bfloat162_rn(silu_mul(g[v].z, u[v].z), silu_mul(g[v].w, u[v].w));
                *reinterpret_cast<uint2*>(a.act + (uint64_t)(q * n_pad + tok[v]) * dc.ff + tl * 128 + 4 * ch[v]) =
                    *reinterpret_cast<uint2*>(o2);
              } else {
                o2[0] = __floats2bfloat162_rn(g[v].x, g[v].y);
                o2[1] = __floats2bfloat162_rn(g[v].z, g[v].w);
                *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(s_dst[tok[v]]) + tl * 128 + 4 * ch[v]) =
                    *reinterpret_cast<uint2*>(o2);
              }
            }
          }
          if (phz == 0) { proxy_fence(); __threadfence(); } else fence_sc(sys);
          epi_bar();
          if (phz == 0) { if (et == 0 && t1 > t0) red_rel_gpu(ctr + kActQ + q, (uint32_t)(t1 - t0)); }
          else if (et >= t0 && et < t1) count_cols(q, et, 128u);
        }
        if (et == 0) { if (phz == 0) CT(7); else CT(10); }
      }
    }
  }
  // ---- teardown: the last CTA to leave resets the launch's counters (stream order makes the
  // next launch see them zeroed)
  tc_fence_before();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(512) : "memory");
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(ctr + 2, 1u) == (uint32_t)(P - 1);
  }
  __syncthreads();
  if (tid == 0) CT(11);
  if (s_last) {
    for (int i = tid; i < a.nq; i += THREADS) ctr[kActQ + i] = 0;
    if (tid == 0) { ctr[0] = 0; ctr[1] = 0; ctr[2] = 0; }
    __threadfence();
  }
}

}  // namespace cold

#ifdef AMOE_COLD_TRACE
extern "C" amoe_status amoe_debug_cold_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, cold::g_cold_trace, sizeof(cold::g_cold_trace)) == cudaSuccess ? AMOE_OK : AMOE_ECUDA;
}
#endif

// Launch the fused cold execution of `nq` queues (qid = l*H + lq, cap = legs to drain at most,
// n_pad = max cap rounded up to 16, <= 128). tm_x / tm_act: the group scratch tile and act
// buffers as TMA maps with {64, n_pad} boxes. Returns launches issued.
int launch_ffn_cold(const DevCtx& c, int nq, const int* qid, const int* cap, int n_pad, const CUtensorMap& tm_x,
                    const CUtensorMap& tm_act, void* tile, void* act, int32_t* qinfo, const CUtensorMap* wmaps,
                    uint32_t seq, int num_sms, cudaStream_t s) {
  using namespace cold;
  static bool attr_done[64] = {false};
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  if (dev_id < 0 || dev_id >= 64) dev_id = 0;
  if (!attr_done[dev_id]) {
    cudaFuncSetAttribute(ffn_cold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DYN);
    attr_done[dev_id] = true;
  }
  ColdArgs a{};
  a.nq = nq;
  a.n_pad = n_pad;
  const int stage_bytes = 2 * A_BYTES + 2 * n_pad * 128;
  a.stages = std::min(MAXS, RING_BUDGET / stage_bytes);
  a.ipt_a = c.d / 64;
  a.ipt_b = c.ff / 128;
  a.ft = c.ff / 128;
  a.dt = c.d / 128;
  a.ia = nq * a.ft * a.ipt_a;
  a.ib = nq * a.dt * a.ipt_b;
  a.seq = seq;
  a.ctr = reinterpret_cast<uint32_t*>(c.peer[c.rank] + c.lay.cold);
  a.part = reinterpret_cast<float*>(c.peer[c.rank] + c.lay.split_part);
  a.qinfo = qinfo;
  a.tile = reinterpret_cast<__nv_bfloat16*>(tile);
  a.act = reinterpret_cast<__nv_bfloat16*>(act);
  a.wmaps = wmaps;
  for (int q = 0; q < nq; ++q) { a.qid[q] = qid[q]; a.cap[q] = cap[q]; }
  // CTAs per phase (Part)
  const int cap_sms = std::min(num_sms, MAXP);
  auto plan = [&](int tiles, int ipt, int32_t& P_, int32_t& s_) {
    // stream-K over every SM: one SM's TMA streams ~40 GB/s of 128-B-row weight boxes, so the
    // HBM needs all of them (a unit = one iteration)
    s_ = ipt;
    P_ = std::min(cap_sms, tiles * ipt);
  };
  plan(nq * a.ft, a.ipt_a, a.pa, a.sa);
  plan(nq * a.dt, a.ipt_b, a.pb, a.sb);
  const int P = std::max(a.pa, a.pb);
  launch_pdl(ffn_cold_kernel, dim3(P), dim3(THREADS), SMEM_DYN, s, tm_x, tm_act, a, c);
  return 1;
}

}  // namespace amoe
