// k_ffn_cold.cu — a4 + a5 + a6 + a7 fused for COLD picks (every queue of the pick holds <= 128
// legs): ONE persistent launch drains the queues, gathers the legs' x rows, runs the SwiGLU
// expert (gate/up, SwiGLU, down) and stores each output row straight into its home's token pool
// (one-sided, NVLink peer store when remote), counting the leg's columns for the merge.
//
// Why (small batches make expert execution weight-loading bound; DESIGN.md
// §5.4): with <= 128 legs per expert the work is streaming the expert's weights (6·d·ff bytes)
// once from HBM — one DeepSeek expert is 17 MB, 2.6 us at HBM speed — so every grid-wide
// hand-off inside the launch is on the critical path. Design, B200-first:
//  * the drain is decided on the host: the scheduler's snapshot gives each queue's consumer head
//    and published depth, so the kernel is told (start, n) and no CTA waits for a device-side
//    drain (CTA 0 only checks the head and advances it);
//  * no grid-wide gather: the token operand of a gate/up K block is gathered by the CTA that
//    needs it (two warps: 16-B loads of the legs' x rows, local or from the home over NVLink,
//    stored into the 128-B-swizzled stage), alongside the weight TMA of the same stage;
//  * the weights of the first ring stages stream before the grid dependency wait (they are
//    constant), so HBM is busy from the first microsecond of the launch;
//  * swap-AB tcgen05 MMA: the weight tile is the M = 128 operand and the legs are N = n_pad
//    (16..128), so a cold expert does not pay a 128-row token tile; gate/up: two MMAs per K
//    step into two TMEM accumulators, SwiGLU in registers; down: two K blocks per stage;
//  * stream-K over weight bytes: CTA c of P_X takes iterations [c·I/P_X, (c+1)·I/P_X) of each
//    phase; a tile split across CTAs is reduced by its LAST arriving CTA (fp32 partials summed
//    in owner order: deterministic), one hand-off instead of a wait on every owner. The host
//    bounds the split so that reduction stays small (launch_ffn_cold);
//  * a down tile waits only for its queue's activations (a counter per queue).
// All CTAs are co-resident (one per SM, grid <= SMs); the only waits are on work that never
// waits itself (gate/up tiles, published ring entries), so the launch cannot deadlock.
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
constexpr int NMAX = 128;             // legs per queue (MMA N, padded to 16)
constexpr int A_BYTES = 128 * 64 * 2; // one 128-row x 64-col bf16 weight box (16 KB)
constexpr int MAXP = 256;             // CTAs (partial slots are indexed by CTA)
constexpr int SMEM_DYN = 219 * 1024;  // dynamic smem request (ring + 1 KB alignment slack)
constexpr int RING_BUDGET = SMEM_DYN - 1024;
constexpr int kPartFloats = NMAX * 256;   // one partial slot: [leg][256] fp32 (128 KB)
// counters (u32, workspace `cold`): [0] exits, then per launch (offsets in ColdArgs):
// [ctr_a + tile] split arrivals of gate/up tiles, [ctr_b + tile] of down tiles, [ctr_act + q]
// gate/up tiles of queue q whose activations are stored

struct ColdArgs {
  int32_t nq, n_pad, stages, stage_bytes;
  int32_t ka, kb;             // K blocks (64 wide) per iteration: gate/up (1, 2), down (1, 2)
  int32_t ipt_a, ipt_b;       // iterations per tile: d/(64·ka) (gate/up), ff/(64·kb) (down)
  int32_t ft, dt;             // tiles per queue: ff/128 (gate/up), d/256 (down: two 128-row halves)
  int32_t ia, ib;             // iterations per phase (all queues)
  int32_t pa, pb;             // CTAs streaming each phase (<= grid)
  int32_t ctr_a, ctr_b, ctr_act;
  uint32_t* ctr;              // workspace counters
  float* part;                // partial slots [(phase*2 + which)*MAXP + cta][kPartFloats]
  int32_t* qinfo;             // out [3*AMOE_MAX_GROUP]: drained n, row offset, ring start per queue
  __nv_bfloat16* act;         // [nq*n_pad][ff]: SwiGLU activations
  const CUtensorMap* wmaps;   // [L*H][3]: 2-D maps (box 64 x 128)
  const CUtensorMap* cmaps;   // [L*H][4]: K-block views W1 x2, W3 x2 (128 rows), W2 x2, W2 x1 (256 rows)
  int32_t qid[AMOE_MAX_GROUP];     // l*H + lq
  int32_t n[AMOE_MAX_GROUP];       // legs to drain (<= NMAX; the scheduler's snapshot depth)
  uint32_t start[AMOE_MAX_GROUP];  // ring position of the first (= the queue's consumer head)
};

// Partition of one phase's iterations (tiles x ipt, one unit = one iteration) over P CTAs:
// CTA c takes [floor(c·I/P), floor((c+1)·I/P)).
struct Part {
  int tiles, ipt, P;
  __device__ __forceinline__ int start(int c) const { return (int)((int64_t)c * (tiles * ipt) / P); }
  // CTA whose range holds iteration it (the largest c with start(c) <= it)
  __device__ __forceinline__ int owner(int it) const {
    const int I = tiles * ipt;
    const int c = (int)(((int64_t)(it + 1) * P - 1) / I);
    return c < P - 1 ? c : P - 1;
  }
};

__device__ __forceinline__ uint32_t ld_acq_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_acqrel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// In-kernel waits are bounded: a wait that has not been satisfied after kWatchdogNs is a bug
// (a dependency that can never complete); the kernel traps instead of hanging the GPU, so the
// launch fails with an error the host sees (cudaErrorLaunchFailure -> AMOE_ECUDA).
constexpr uint64_t kWatchdogNs = 4000000000ull;
__device__ __noinline__ void watchdog_trap(uint32_t where) {
  printf("amoe cold kernel watchdog: block %d thread %d wait %u\n", blockIdx.x, threadIdx.x, where);
  asm volatile("trap;");
}
// The TMA producer observes dependencies with acquire LOADS, never a fence: a fence would wait
// for the thread's outstanding bulk copies and drain the weight pipeline.
// Every CTA's producer may poll the same counter: a short sleep between polls keeps ~150 pollers
// from crowding the counter's L2 line while its writers' release-adds queue behind them.
__device__ __forceinline__ void spin_until_eq_acq(const uint32_t* p, uint32_t v, uint32_t where) {
  if (ld_acq_gpu(p) == v) return;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t i = 1;; ++i) {
    __nanosleep(64);
    if (ld_acq_gpu(p) == v) return;
    if ((i & 1023u) == 0 && globaltimer_ns() - t0 > kWatchdogNs) watchdog_trap(where);
  }
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
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
// a published ring entry (seq = position + 1, release-stored last by its producer)
__device__ __forceinline__ amoe_leg wait_leg(const amoe_leg* ring, uint32_t mask, uint32_t pos) {
  const amoe_leg* e = ring + (pos & mask);
  if (ld_acquire(&e->seq) != pos + 1u) {
    const uint64_t t0 = globaltimer_ns();
    for (uint32_t i = 1; ld_acquire(&e->seq) != pos + 1u; ++i)
      if ((i & 255u) == 0 && globaltimer_ns() - t0 > kWatchdogNs) watchdog_trap(9);
  }
  return *e;
}
// generic-proxy stores -> visible to async-proxy (TMA / tensor core) reads
__device__ __forceinline__ void proxy_fence_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }   // warps 4..7

// The CTA's j-th item (phase A items first, then phase B).
struct Items {
  int a0, a1, b0, b1, ipt_a, ipt_b;
  __device__ __forceinline__ int count() const { return (a1 - a0) + (b1 - b0); }
  __device__ __forceinline__ void get(int j, int& phase, int& tile, int& k) const {
    if (j < a1 - a0) { const int it = a0 + j; phase = 0; tile = it / ipt_a; k = it - tile * ipt_a; }
    else { const int it = b0 + j - (a1 - a0); phase = 1; tile = it / ipt_b; k = it - tile * ipt_b; }
  }
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

// partial slot of CTA o's segment in tile t: 0 when o's range starts inside t (its first
// segment of the phase, k0 > 0), else 1 (a segment starting at the tile's first iteration)
__device__ __forceinline__ int which_of(int o, int t, const Part& pt) { return pt.start(o) > t * pt.ipt ? 0 : 1; }

#ifdef AMOE_COLD_TRACE
// diagnostic build only: per-CTA globaltimer stamps of the last launch (tools/cold_trace.py)
__device__ unsigned long long g_cold_trace[16][MAXP];
#define CT(i) (g_cold_trace[i][blockIdx.x] = globaltimer_ns())
// accumulated wait time (ns) of one role, rows 12..15
#define CW_BEGIN() const uint64_t cw_t0 = globaltimer_ns()
#define CW_END(i) (g_cold_trace[i][blockIdx.x] += globaltimer_ns() - cw_t0)
#else
#define CT(i) ((void)0)
#define CW_BEGIN() ((void)0)
#define CW_END(i) ((void)0)
#endif

__global__ void __launch_bounds__(THREADS, 1)
ffn_cold_kernel(const __grid_constant__ CUtensorMap tmAct, const __grid_constant__ ColdArgs a,
                const __grid_constant__ DevCtx dc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (threadIdx.x == 0) CT(0);
  __shared__ uint64_t bars[2 * MAXS + 4];      // full[MAXS], empty[MAXS], tfull[2], tempty[2]
  __shared__ uint32_t tmem_holder[4];
  __shared__ amoe_leg s_leg[NMAX];             // legs of queue s_legq (epilogue: down destinations)
  __shared__ int s_legq;
  __shared__ __align__(16) __nv_bfloat16 s_stage[16][128];   // epilogue transpose (16 legs)
  __shared__ int s_last;
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = gridDim.x, cta = blockIdx.x;
  const int n_pad = a.n_pad, S = a.stages;
  const int stage_bytes = a.stage_bytes;
  const int KA = a.ka, KB = a.kb;
  const Part part_a{a.ia / a.ipt_a, a.ipt_a, a.pa}, part_b{a.ib / a.ipt_b, a.ipt_b, a.pb};
  const bool in_a = cta < a.pa, in_b = cta < a.pb;
  const Items it{in_a ? part_a.start(cta) : 0, in_a ? part_a.start(cta + 1) : 0, in_b ? part_b.start(cta) : 0,
                 in_b ? part_b.start(cta + 1) : 0, a.ipt_a, a.ipt_b};
  const int n_items = it.count();
  uint32_t* ctr = a.ctr;

  if (tid == 0) {
    // full: the producer's expect_tx arrive + one cp.async completion arrive per gather lane
    // (phase B: the producer arrives for them); empty / tfull: one MMA commit; tempty: one
    // epilogue arrive
    for (int s = 0; s < S; ++s) { mbar_init(smem_u32(&bars[s]), 1 + 64); mbar_init(smem_u32(&bars[MAXS + s]), 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(smem_u32(&bars[2 * MAXS + b]), 1); mbar_init(smem_u32(&bars[2 * MAXS + 2 + b]), 1); }
    s_legq = -1;
#ifdef AMOE_COLD_TRACE
    for (int i = 12; i < 16; ++i) g_cold_trace[i][blockIdx.x] = 0;
    g_cold_trace[9][blockIdx.x] = 0;
#endif
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
      // ===================== TMA producer: weights of every item; the activation operand of
      // down items once their queue's gate/up tiles are all stored
      const uint64_t wpol = policy_evict_first();
      auto issue_a = [&](int j, int s) {
        int ph, t, k;
        it.get(j, ph, t, k);
        const uint32_t sa = smem_u32(ring + s * stage_bytes);
        const uint32_t full = smem_u32(&bars[s]);
        // stage: gate/up: W1 [KA][128][64], W3 [KA][128][64], legs [KA][n_pad][64];
        //        down:    W2 [KB][256][64] (two 128-row halves per K block), act [KB][n_pad][64]
        if (ph == 0) {
          mbar_expect_tx(full, 2 * KA * A_BYTES);
          const int q = t / a.ft, f = t - q * a.ft;
          if (KA == 1) {
            const CUtensorMap* wm = a.wmaps + a.qid[q] * 3;
            tma_load_2d_hint(sa, wm, k * 64, f * 128, full, wpol);
            tma_load_2d_hint(sa + A_BYTES, wm + 1, k * 64, f * 128, full, wpol);
          } else {
            const CUtensorMap* cm = a.cmaps + a.qid[q] * 4;
            tma_load_3d_hint(sa, cm, 0, f * 128, KA * k, full, wpol);
            tma_load_3d_hint(sa + KA * A_BYTES, cm + 1, 0, f * 128, KA * k, full, wpol);
          }
        } else {
          mbar_expect_tx(full, KB * (2 * A_BYTES + n_pad * 128));
          mbar_arrive_cnt(full, 64);                  // the gather lanes' share (no gather here)
          const int q = t / a.dt, dtl = t - q * a.dt;
          const CUtensorMap* cm = a.cmaps + a.qid[q] * 4 + (KB == 2 ? 2 : 3);
          tma_load_3d_hint(sa, cm, 0, dtl * 256, KB * k, full, wpol);
        }
      };
      int ready_q = -1;                               // queue whose activations are all stored
      auto issue_act = [&](int j, int s) {
        int ph, t, k;
        it.get(j, ph, t, k);
        const int q = t / a.dt;
        if (q != ready_q) {
          spin_until_eq_acq(ctr + a.ctr_act + q, (uint32_t)a.ft, 6);
          proxy_fence_global();
          ready_q = q;
        }
        const uint32_t sb = smem_u32(ring + s * stage_bytes) + KB * 2 * A_BYTES;
        const uint32_t full = smem_u32(&bars[s]);
        tma_load_3d(sb, &tmAct, 0, q * n_pad, KB * k, full);
      };
      // the weight tensor maps live in the workspace (global memory): prefetch the ones this CTA's
      // items use into the descriptor cache before the first loads
      if (n_items > 0) {
        int ph, t, k;
        it.get(0, ph, t, k);
        int q0 = ph == 0 ? t / a.ft : t / a.dt;
        it.get(n_items - 1, ph, t, k);
        int q1 = ph == 0 ? t / a.ft : t / a.dt;
        if (it.a1 > it.a0 && it.b1 > it.b0) { q0 = 0; q1 = a.nq - 1; }
        for (int q = q0; q <= q1 && q < q0 + 8; ++q) {
          const CUtensorMap* cm = a.cmaps + a.qid[q] * 4;
          if (KA == 1) { tma_prefetch(a.wmaps + a.qid[q] * 3); tma_prefetch(a.wmaps + a.qid[q] * 3 + 1); }
          else { tma_prefetch(cm); tma_prefetch(cm + 1); }
          tma_prefetch(cm + (KB == 2 ? 2 : 3));
        }
        tma_prefetch(&tmAct);
      }
      // weights of the first stages stream before the grid dependency (they are constant)
      int stage = 0;
      uint32_t phase = 0;
      int j = 0;
      int pend[MAXS], ps[MAXS], np = 0, ph0 = 0;     // down items whose act load is pending
      for (; j < n_items && j < S; ++j) {
        issue_a(j, stage);
        int ph, t, k;
        it.get(j, ph, t, k);
        if (ph == 1) { pend[(ph0 + np) % MAXS] = j; ps[(ph0 + np) % MAXS] = stage; ++np; }
        if (++stage == S) { stage = 0; phase ^= 1u; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      CT(1);
      for (;;) {
        // act loads of pending down items, in order: blocking only when every stage waits for
        // its act or nothing is left to prefetch, else polled between weight issues
        while (np > 0) {
          int ph, t, k;
          it.get(pend[ph0], ph, t, k);
          const int q = t / a.dt;
          const bool stuck = np == S || j >= n_items;
          if (q != ready_q && !stuck && ld_acq_gpu(ctr + a.ctr_act + q) != (uint32_t)a.ft) break;
          issue_act(pend[ph0], ps[ph0]);
          ph0 = (ph0 + 1) % MAXS; --np;
        }
        if (j >= n_items) {
          if (np == 0) break;
          continue;
        }
        if (np > 0 && np < S) {
          // poll: a free stage takes the next item's weights; otherwise re-check the act
          uint32_t ok;
          asm volatile("{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                       : "=r"(ok) : "r"(smem_u32(&bars[MAXS + stage])), "r"(phase ^ 1u) : "memory");
          if (!ok) continue;
        }
        {
          CW_BEGIN();
          mbar_wait_wd(smem_u32(&bars[MAXS + stage]), phase ^ 1u, 1);
          CW_END(12);
        }
        issue_a(j, stage);
        {
          int ph, t, k;
          it.get(j, ph, t, k);
          if (ph == 1) { pend[(ph0 + np) % MAXS] = j; ps[(ph0 + np) % MAXS] = stage; ++np; }
        }
        ++j;
        if (++stage == S) { stage = 0; phase ^= 1u; }
      }
      CT(2);
    }
  } else if (warp == 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0) {
      // ===================== MMA issuer (single thread): swap-AB, D[128 weight rows][n_pad legs]
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int j = 0; j < n_items; ++j) {
        int ph, t, k;
        it.get(j, ph, t, k);
        const bool first = it.seg_first(j), last = it.seg_last(j);
        if (first) {
          CW_BEGIN();
          mbar_wait_wd(smem_u32(&bars[2 * MAXS + 2 + acc]), acc_phase ^ 1u, 2);
          CW_END(9);
          tc_fence_after();
        }
        const uint32_t d0 = tmem_base + (uint32_t)(acc * 256);
        {
          CW_BEGIN();
          mbar_wait_wd(smem_u32(&bars[stage]), phase, 3);
          CW_END(13);
        }
        tc_fence_after();
#ifndef AMOE_COLD_NOPROXY   // diagnostic only
        if (ph == 0) proxy_fence_smem();   // the gathered leg rows (cp.async, generic proxy) -> tensor core
#endif
        const uint32_t sa = smem_u32(ring + stage * stage_bytes);
#ifdef AMOE_COLD_NOMMA   // diagnostic only: wrong results
        if (false) {
#else
        if (ph == 0) {
#endif
          for (int kb = 0; kb < KA; ++kb) {
            const uint64_t a0d = umma_desc_sw128(sa + kb * A_BYTES), a1d = umma_desc_sw128(sa + (KA + kb) * A_BYTES);
            const uint64_t b0d = umma_desc_sw128(sa + 2 * KA * A_BYTES + kb * n_pad * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t accum = (!first || kb > 0 || kk > 0) ? 1u : 0u;
              umma_bf16(d0, a0d + 2 * kk, b0d + 2 * kk, idesc, accum);                    // gate
              umma_bf16(d0 + (uint32_t)n_pad, a1d + 2 * kk, b0d + 2 * kk, idesc, accum);  // up
            }
          }
        } else
#ifdef AMOE_COLD_NOMMA
        if (false)
#endif
        {
          for (int kb = 0; kb < KB; ++kb) {
            // rows 0..127 and 128..255 of the 256-row W2 slab into the two accumulator halves
            const uint64_t a0d = umma_desc_sw128(sa + kb * 2 * A_BYTES), a1d = umma_desc_sw128(sa + kb * 2 * A_BYTES + A_BYTES);
            const uint64_t b0d = umma_desc_sw128(sa + KB * 2 * A_BYTES + kb * n_pad * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t accum = (!first || kb > 0 || kk > 0) ? 1u : 0u;
              umma_bf16(d0, a0d + 2 * kk, b0d + 2 * kk, idesc, accum);
              umma_bf16(d0 + (uint32_t)n_pad, a1d + 2 * kk, b0d + 2 * kk, idesc, accum);
            }
          }
        }
        umma_commit(smem_u32(&bars[MAXS + stage]));
        if (++stage == S) { stage = 0; phase ^= 1u; }
        if (last) {
          umma_commit(smem_u32(&bars[2 * MAXS + acc]));
          if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        }
      }
      CT(3);
    }
  } else if (warp == 2 || warp == 3) {
    // ===================== gather warps: the leg rows of each gate/up item's K block, straight
    // from the legs' x rows (local, or from the home over NVLink) into the swizzled stage
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int gw = warp - 2;                     // rows [gw*64, gw*64 + 64)
    // lane's chunks: u = 0..15 -> row 4u + lane/8 of this warp's 64, 16-B chunk lane % 8 of the
    // K block's 128 B, copied with cp.async; each lane's copies of a stage arrive on its full
    // barrier when they land (cp.async.mbarrier.arrive.noinc), so the warp never waits for them
    // (the MMA thread orders them for the tensor core with a proxy fence)
    constexpr int MAXC = 16;
    int cur_q = -1;
    const char* rp[MAXC];                        // source row of chunk u (x row of the leg)
#pragma unroll
    for (int u = 0; u < MAXC; ++u) rp[u] = nullptr;
    int nq_rows = 0;
    int stage = 0;
    uint32_t phase = 0;
    const int na = it.a1 - it.a0;
    for (int j = 0; j < na; ++j) {
      int ph, t, k;
      it.get(j, ph, t, k);
      const int q = t / a.ft;
      if (q != cur_q) {
        cur_q = q;
        const int n = a.n[q];
        nq_rows = min(64, max(0, n - gw * 64));
        const amoe_leg* rg = ring_ptr(dc, dc.rank, a.qid[q]);
        const char* src0 = nullptr;              // x row of leg (gw*64 + lane)
        const char* src1 = nullptr;              // x row of leg (gw*64 + 32 + lane)
        auto src_of = [&](int i) -> const char* {
          const amoe_leg e = wait_leg(rg, dc.ring_mask, a.start[q] + (uint32_t)i);
          int home = e.home, slot = e.token_slot;
          if (home < 0 || home >= dc.G || slot < 0 || slot >= dc.T) {
            raise_fault(dc, F_STALE_ENTRY, (uint32_t)a.qid[q], a.start[q] + (uint32_t)i, e.seq);
            home = dc.rank; slot = 0;
          }
          return reinterpret_cast<const char*>(dc.peer[home] + dc.lay.x) + (uint64_t)slot * dc.d * 2;
        };
        if (lane < nq_rows) src0 = src_of(gw * 64 + lane);
        if (lane + 32 < nq_rows) src1 = src_of(gw * 64 + 32 + lane);
#pragma unroll
        for (int u = 0; u < MAXC; ++u) {
          const int r = 4 * u + (lane >> 3);
          const uintptr_t p0 = __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src0), r & 31);
          const uintptr_t p1 = __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src1), r & 31);
          rp[u] = reinterpret_cast<const char*>(r < 32 ? p0 : p1) + (lane & 7) * 16;
        }
        if (lane == 0 && j == 0) CT(4);
      }
      {
        CW_BEGIN();
        mbar_wait_wd(smem_u32(&bars[MAXS + stage]), phase ^ 1u, 10);
        if (lane == 0 && gw == 0) CW_END(14);
      }
      // chunk c of row i of K block kb lands at byte kb*n_pad*128 + i*128 + ((c ^ (i & 7)) * 16)
      const uint32_t sb = smem_u32(ring + stage * stage_bytes + 2 * KA * A_BYTES);
      for (int kb = 0; kb < KA; ++kb) {
#pragma unroll
        for (int u = 0; u < MAXC; ++u) {
          const int r = 4 * u + (lane >> 3), c = lane & 7, i = gw * 64 + r;
#ifdef AMOE_COLD_NOGATHER   // diagnostic only: wrong results
          if (false)
#else
          if (r < nq_rows)
#endif
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                         :: "r"(sb + kb * n_pad * 128 + i * 128 + ((c ^ (i & 7)) * 16)),
                            "l"(rp[u] + (uint64_t)(KA * k + kb) * 128) : "memory");
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(smem_u32(&bars[stage])) : "memory");
      if (++stage == S) { stage = 0; phase ^= 1u; }
    }
  } else {
    // ===================== epilogue (warps 4..7): TMEM lane quarter ew, weight row r
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int ew = warp - 4, r = ew * 32 + lane, et = tid - 128;
    const bool sys = dc.G > 1;
    if (cta == 0 && warp == 7) {
      // the drain's bookkeeping (a4): check each queue's consumer head is the position the
      // scheduler saw, advance it past the n drained legs, publish (n, row offset, start), count
      uint32_t tot = 0;
      for (int q = lane; q < a.nq; q += 32) {
        uint32_t* qc = qctr_ptr(dc, dc.rank, a.qid[q]);
        const uint32_t head = qc[2];
        if (head != a.start[q]) raise_fault(dc, F_HEAD_MISMATCH, (uint32_t)a.qid[q], a.start[q], head);
        qc[2] = a.start[q] + (uint32_t)a.n[q];
        a.qinfo[q] = a.n[q];
        a.qinfo[AMOE_MAX_GROUP + q] = q * n_pad;
        a.qinfo[2 * AMOE_MAX_GROUP + q] = (int32_t)a.start[q];
        tot += (uint32_t)a.n[q];
      }
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      if (lane == 0) atomicAdd(wsp<unsigned long long>(dc, dc.rank, dc.lay.stats) + 2, (unsigned long long)tot);
      if (dc.xlog) {
        // checked mode: one record per nonempty queue + its legs (seq := the token's pass)
        uint32_t* xl = dc.xlog;
        for (int q = 0; q < a.nq; ++q) {
          const uint32_t n = (uint32_t)a.n[q], head = a.start[q];
          if (!n) continue;
          uint32_t e0 = 0, l0 = 0;
          if (lane == 0) {
            e0 = atomicAdd(xl + 0, 1u);
            l0 = atomicAdd(xl + 1, n);
            if (e0 < xl[2]) {
              uint32_t* rec = xlog_exec(xl) + 4 * (uint64_t)e0;
              rec[0] = (uint32_t)a.qid[q]; rec[1] = head; rec[2] = n; rec[3] = l0;
            }
          }
          l0 = __shfl_sync(0xffffffffu, l0, 0);
          const amoe_leg* rg = ring_ptr(dc, dc.rank, a.qid[q]);
          for (uint32_t i = lane; i < n; i += 32) {
            if (l0 + i >= xl[3]) break;
            amoe_leg e = wait_leg(rg, dc.ring_mask, head + i);
            const int home = (e.home >= 0 && e.home < dc.G) ? e.home : dc.rank;
            const int slot = (e.token_slot >= 0 && e.token_slot < dc.T) ? e.token_slot : 0;
            e.seq = (uint32_t)reinterpret_cast<const int32_t*>(dc.peer[home] + dc.lay.tok_pass)[slot];
            xlog_legs(xl)[l0 + i] = e;
          }
          __syncwarp();
        }
      }
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    // legs of queue q (down destinations), cached in smem
    auto load_legs = [&](int q) {
      if (s_legq == q) return;
      epi_bar();
      if (et < a.n[q]) s_leg[et] = wait_leg(ring_ptr(dc, dc.rank, a.qid[q]), dc.ring_mask, a.start[q] + (uint32_t)et);
      epi_bar();
      if (et == 0) s_legq = q;
      epi_bar();
    };
    auto dst_row = [&](int i) -> __nv_bfloat16* {
      const amoe_leg& e = s_leg[i];
      return reinterpret_cast<__nv_bfloat16*>(dc.peer[e.home] + dc.lay.pool) +
             ((uint64_t)e.token_slot * dc.KS + (uint64_t)e.k) * dc.d;
    };
    // a down tile's 128 columns of every leg stored: count them (+ the remote legs, once per leg)
    auto count_legs = [&](int q, int tl) {
      if (et < a.n[q]) {
        const amoe_leg& e = s_leg[et];
        leg_pieces_done(dc, e.home, e.token_slot, e.k, 256u);
      }
      if (tl == 0) {
        const uint32_t rem = __popc(__ballot_sync(0xffffffffu, et < a.n[q] && s_leg[et].home != dc.rank));
        if (lane == 0 && rem)
          atomicAdd(wsp<unsigned long long>(dc, dc.rank, dc.lay.stats) + 3, (unsigned long long)rem);
      }
    };
    int j = 0;
    for (int phz = 0; phz < 2; ++phz) {
      const int jend = phz == 0 ? (it.a1 - it.a0) : n_items;
      const int ipt = phz == 0 ? a.ipt_a : a.ipt_b;
      const Part& pt = phz == 0 ? part_a : part_b;
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
        if (et == 0) mbar_wait_wd(tfull, acc_phase, 4);
        epi_bar();
        tc_fence_after();
        const uint32_t tb = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(ew * 32) << 16);
        const int q = ph == 0 ? t / a.ft : t / a.dt;
        const int tl = ph == 0 ? t - q * a.ft : t - q * a.dt;
        const int n = a.n[q];
        const bool whole = k0 == 0 && k1 == ipt;
        if (ph == 1) load_legs(q);
        const int which = k0 > 0 ? 0 : 1;
        float* part = a.part + (size_t)((ph * 2 + which) * MAXP + cta) * kPartFloats;
        for (int c0 = 0; c0 < n; c0 += 16) {
          float v[32];
          // v[0..16): gate (gate/up) or output rows 0..127 (down); v[16..32): up, or rows 128..255
          tmem_ld16x2(tb + c0, tb + n_pad + c0, v);
          const int m = min(16, n - c0);
          if (whole) {
            // thread r holds column r of 16 leg rows: transpose through smem, then every row
            // (256 B: 128 columns) leaves as 16-B vector stores; down tiles store two halves
            for (int half = 0; half < (ph == 0 ? 1 : 2); ++half) {
              for (int i = 0; i < m; ++i)
                s_stage[i][r] = __float2bfloat16_rn(ph == 0 ? silu_mul(v[i], v[16 + i]) : v[16 * half + i]);
              epi_bar();
              for (int x = et; x < m * 16; x += 128) {
                const int tk = x >> 4, cc = x & 15;
                const uint4 val = reinterpret_cast<const uint4*>(s_stage[tk])[cc];
                __nv_bfloat16* dst = ph == 0 ? a.act + (uint64_t)(q * n_pad + c0 + tk) * dc.ff + tl * 128
                                             : dst_row(c0 + tk) + tl * 256 + half * 128;
                reinterpret_cast<uint4*>(dst)[cc] = val;
              }
              epi_bar();
            }
          } else {
            for (int i = 0; i < m; ++i) {
              float* row = part + (size_t)(c0 + i) * 256;
              row[r] = v[i];
              row[128 + r] = v[16 + i];
            }
          }
        }
        tc_fence_before();
        epi_bar();
        if (et == 0) mbar_arrive(tempty);        // TMEM buffer free for the MMA
        if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        bool finish = whole;
        if (!whole) {
          // split tile: publish this partial; the last of the tile's owners to arrive sums all
          // of them (owner order: deterministic) and finishes the tile
          __threadfence();
          epi_bar();
          if (et == 0) {
            const int first = pt.owner(t * ipt), lastc = pt.owner(t * ipt + ipt - 1);
            const uint32_t old = atom_acqrel_gpu(ctr + (ph == 0 ? a.ctr_a : a.ctr_b) + t, 1u);
            s_last = old == (uint32_t)(lastc - first);
          }
          epi_bar();
          if (s_last) {
            if (et == 0) CT(ph == 0 ? 5 : 6);
            __threadfence();
            const int first = pt.owner(t * ipt), lastc = pt.owner(t * ipt + ipt - 1);
            const int items = n * 32;                // (leg, 4-row chunk)
            // two items per thread per pass, the owners' partials loaded 4 at a time for both
            // (16 loads in flight), then summed in owner order
            for (int x0 = et; x0 < items; x0 += 256) {
              const int x1 = x0 + 128;
              const bool ok1 = x1 < items;
              const int tk0 = x0 >> 5, ch0 = x0 & 31, tk1 = x1 >> 5, ch1 = x1 & 31;
              float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), u0 = g0, g1 = g0, u1 = g0;
              for (int ob = first; ob <= lastc; ob += 4) {
                float4 pg0[4], pu0[4], pg1[4], pu1[4];
#pragma unroll
                for (int i2 = 0; i2 < 4; ++i2)
                  if (ob + i2 <= lastc) {
                    const float* slot = a.part + (size_t)((ph * 2 + which_of(ob + i2, t, pt)) * MAXP + ob + i2) * kPartFloats;
                    const float* r0 = slot + (size_t)tk0 * 256 + 4 * ch0;
                    pg0[i2] = __ldcg(reinterpret_cast<const float4*>(r0));
                    pu0[i2] = __ldcg(reinterpret_cast<const float4*>(r0 + 128));
                    if (ok1) {
                      const float* r1 = slot + (size_t)tk1 * 256 + 4 * ch1;
                      pg1[i2] = __ldcg(reinterpret_cast<const float4*>(r1));
                      pu1[i2] = __ldcg(reinterpret_cast<const float4*>(r1 + 128));
                    }
                  }
#pragma unroll
                for (int i2 = 0; i2 < 4; ++i2)
                  if (ob + i2 <= lastc) {
                    g0.x += pg0[i2].x; g0.y += pg0[i2].y; g0.z += pg0[i2].z; g0.w += pg0[i2].w;
                    u0.x += pu0[i2].x; u0.y += pu0[i2].y; u0.z += pu0[i2].z; u0.w += pu0[i2].w;
                    if (ok1) {
                      g1.x += pg1[i2].x; g1.y += pg1[i2].y; g1.z += pg1[i2].z; g1.w += pg1[i2].w;
                      u1.x += pu1[i2].x; u1.y += pu1[i2].y; u1.z += pu1[i2].z; u1.w += pu1[i2].w;
                    }
                  }
              }
#pragma unroll
              for (int vv = 0; vv < 2; ++vv) {
                if (vv == 1 && !ok1) break;
                const float4 g = vv ? g1 : g0, u = vv ? u1 : u0;
                const int tok = vv ? tk1 : tk0, ch = vv ? ch1 : ch0;
                __nv_bfloat162 o2[2];
                if (ph == 0) {
                  o2[0] = __floats2bfloat162_rn(silu_mul(g.x, u.x), silu_mul(g.y, u.y));
                  o2[1] = __floats2bfloat162_rn(silu_mul(g.z, u.z), silu_mul(g.w, u.w));
                  *reinterpret_cast<uint2*>(a.act + (uint64_t)(q * n_pad + tok) * dc.ff + tl * 128 + 4 * ch) =
                      *reinterpret_cast<uint2*>(o2);
                } else {
                  __nv_bfloat16* drow = dst_row(tok) + tl * 256 + 4 * ch;
                  o2[0] = __floats2bfloat162_rn(g.x, g.y);
                  o2[1] = __floats2bfloat162_rn(g.z, g.w);
                  *reinterpret_cast<uint2*>(drow) = *reinterpret_cast<uint2*>(o2);
                  o2[0] = __floats2bfloat162_rn(u.x, u.y);
                  o2[1] = __floats2bfloat162_rn(u.z, u.w);
                  *reinterpret_cast<uint2*>(drow + 128) = *reinterpret_cast<uint2*>(o2);
                }
              }
            }
            finish = true;
          }
        }
        if (finish) {
          // publish the finished tile: gate/up -> the act counter of its queue (the down tiles'
          // TMA reads them); down -> the leg columns of every leg
          if (ph == 0) { proxy_fence_global(); __threadfence(); }
          else fence_sc(sys);
          epi_bar();
          if (ph == 0) { if (et == 0) red_rel_gpu(ctr + a.ctr_act + q, 1u); }
          else count_legs(q, tl);
        }
      }
      if (et == 0) CT(phz == 0 ? 7 : 8);
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
    s_last = atomicAdd(ctr + 0, 1u) == (uint32_t)(P - 1);
  }
  __syncthreads();
  if (tid == 0) CT(11);
  if (s_last) {
    const int nctr = a.ctr_act + a.nq;
    for (int i = 1 + tid; i < nctr; i += THREADS) ctr[i] = 0;
    if (tid == 0) ctr[0] = 0;
    __threadfence();
  }
}

}  // namespace cold

#ifdef AMOE_COLD_TRACE
extern "C" amoe_status amoe_debug_cold_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, cold::g_cold_trace, sizeof(cold::g_cold_trace)) == cudaSuccess ? AMOE_OK : AMOE_ECUDA;
}
#endif

// Launch the fused cold execution of `nq` queues (qid = l*H + lq): queue q drains exactly n[q]
// (<= 128) legs from ring position start[q] (its consumer head). n_pad = max n rounded up to 16.
// tm_act: the group act buffer as a TMA map with a {64, n_pad} box. Returns launches issued, or
// -1 when the counters would not fit.
// K blocks per iteration (ka: gate/up, kb: down): the deepest that keeps >= 3 ring stages and
// divides the K extents (d / 64, ff / 64). Deeper iterations mean fewer TMA boxes per byte.
void cold_blocks(int d, int ff, int n_pad, int* ka, int* kb) {
  using namespace cold;
  if (const char* e = getenv("AMOE_COLD_KAKB")) {   // A/B override "ka,kb" (profiles/r02_cold_sweep.md)
    int x = 0, y = 0;
    if (sscanf(e, "%d,%d", &x, &y) == 2 && (x == 1 || x == 2) && (y == 1 || y == 2) && (d / 64) % x == 0 &&
        (ff / 64) % y == 0) {
      *ka = x;
      *kb = y;
      return;
    }
  }
  const int cand[4][2] = {{2, 2}, {1, 2}, {2, 1}, {1, 1}};
  for (const auto& ck : cand) {
    const int sb = std::max(ck[0] * (2 * A_BYTES + n_pad * 128), ck[1] * (2 * A_BYTES + n_pad * 128));
    if ((d / 64) % ck[0] || (ff / 64) % ck[1] || RING_BUDGET / sb < 3) continue;
    *ka = ck[0];
    *kb = ck[1];
    return;
  }
  *ka = 1;
  *kb = 1;
}

int launch_ffn_cold(const DevCtx& c, int nq, const int* qid, const int* n, const uint32_t* start, int n_pad, int ka,
                    int kb, const CUtensorMap& tm_act, void* act, int32_t* qinfo, const CUtensorMap* wmaps,
                    const CUtensorMap* cmaps, int num_sms, cudaStream_t s) {
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
  a.ka = ka;
  a.kb = kb;
  a.stage_bytes = std::max(ka * (2 * A_BYTES + n_pad * 128), kb * (2 * A_BYTES + n_pad * 128));
  a.stages = std::min(MAXS, RING_BUDGET / a.stage_bytes);
  if (a.stages < 2) return -1;
  a.ipt_a = c.d / (64 * ka);
  a.ipt_b = c.ff / (64 * kb);
  a.ft = c.ff / 128;
  a.dt = c.d / 256;
  const int tiles_a = nq * a.ft, tiles_b = nq * a.dt;
  a.ia = tiles_a * a.ipt_a;
  a.ib = tiles_b * a.ipt_b;
  a.ctr_a = 16;
  a.ctr_b = a.ctr_a + tiles_a;
  a.ctr_act = a.ctr_b + tiles_b;
  if (a.ctr_act + nq > kColdCtr) return -1;
  a.ctr = reinterpret_cast<uint32_t*>(c.peer[c.rank] + c.lay.cold);
  a.part = reinterpret_cast<float*>(c.peer[c.rank] + c.lay.split_part);
  a.qinfo = qinfo;
  a.act = reinterpret_cast<__nv_bfloat16*>(act);
  a.wmaps = wmaps;
  a.cmaps = cmaps;
  for (int q = 0; q < nq; ++q) { a.qid[q] = qid[q]; a.n[q] = n[q]; a.start[q] = start[q]; }
  // CTAs per phase: stream-K over every SM (one SM's TMA streams a few tens of GB/s of weight
  // boxes, so HBM needs all of them), except that a split tile is reduced by one CTA reading
  // every owner's partial: the split is bounded so that read stays <= kRedBytes per tile
  // (AMOE_COLD_RED_KB overrides; A/B in profiles/r02_cold_sweep.md)
  static int red_kb = -1;
  if (red_kb < 0) {
    const char* e = getenv("AMOE_COLD_RED_KB");
    red_kb = e ? std::max(1, atoi(e)) : 64;
  }
  const int cap_sms = std::min(num_sms, MAXP);
  auto plan = [&](int tiles, int ipt, int width) {
    // long tiles (>= 32 iterations: Mixtral's gate/up and down) make every segment a large
    // stream of weights next to which a partial is small: split freely over every SM. Short
    // tiles (DeepSeek) bound the split by the partial bytes the last arriver reads
    if (ipt >= 32) return std::min(cap_sms, tiles * ipt);
    const int64_t part_bytes = (int64_t)n_pad * width * 4;
    const int max_seg = (int)std::max<int64_t>(1, ((int64_t)red_kb << 10) / part_bytes);
    // nseg <= ceil(ipt·P/I) + 1, so P <= tiles·(max_seg - 1) keeps every tile within max_seg
    int64_t p = (int64_t)tiles * std::max(1, max_seg - 1);
    p = std::max<int64_t>(p, std::min<int64_t>(tiles, cap_sms));
    return (int)std::min<int64_t>({(int64_t)cap_sms, (int64_t)tiles * ipt, p});
  };
  a.pa = plan(tiles_a, a.ipt_a, 256);
  a.pb = plan(tiles_b, a.ipt_b, 256);
  const int P = std::max(a.pa, a.pb);
  launch_pdl(ffn_cold_kernel, dim3(P), dim3(THREADS), SMEM_DYN, s, tm_act, a, c);
  return 1;
}

}  // namespace amoe
