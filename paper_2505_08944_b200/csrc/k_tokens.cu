// k_tokens.cu — token-side kernels of the AEP hot path (home rank):
//   token_init  : admit tokens (h, x = rmsnorm(h), state)                     (reading c7)
//   enqueue     : a1 router top-K + a2 scatter of the K legs into µ-queues
//   cdrain      : snapshot of the combine ring (token pool readiness, L228)
//   combine     : a8 weighted top-K merge + RMSNorm + relabel + fused a1/a2     (L175, L209, L228, L236)
//   announce    : multi-GPU quiescence flag
#include "amoe_internal.cuh"

namespace amoe {

constexpr int kTokThreads = 256;
constexpr int kTokWarps = kTokThreads / kWarp;
#ifndef AMOE_TPW
#define AMOE_TPW 4
#endif
constexpr int kTPW = AMOE_TPW;                // tokens per warp per chunk
constexpr int kTPC = kTokWarps * kTPW;        // tokens per CTA chunk
// 16-byte chunks per lane batched in the merge. 1 keeps the kernel at ~48 registers (~40 resident
// warps/SM); measured on B200: kU = 4 (128 regs) and kU = 2 with a register cap (spills) were
// both slower (Mixtral combine 225 -> 268 -> 458 us/layer): parallelism comes from warps.
constexpr int kU = 1;

// Tokens one CTA takes per chunk of an n-token launch: kTPC (kTPW per warp) when the grid has
// that much work, else a multiple of the warp count spread over the grid so a warp merges at most
// one token — a small merge is one latency chain per token, not kTPW of them in a row (the
// combine after a cold pick of a few dozen tokens: profiles/r02_combine_small.md).
__device__ __forceinline__ int chunk_tokens(int n) {
  int tpc = (n + (int)gridDim.x - 1) / (int)gridDim.x;
  tpc = (tpc + kTokWarps - 1) / kTokWarps * kTokWarps;
  return tpc < kTokWarps ? kTokWarps : (tpc > kTPC ? kTPC : tpc);
}

struct PendingLeg {
  int32_t r;      // owner rank (-1 = inactive)
  int32_t q;      // queue index on the owner
  amoe_leg g;
};

// ---------------------------------------------------------------------------- routing (a1)
// Warp-cooperative top-K of z[0..E) (ties -> lower expert index) and softmax over the K
// selected logits. Split in two so callers can issue the logit loads early: route_load reads
// lane's share of z (expert lane + 32 j), route_select returns, in lane k < K, the k-th expert
// and its weight (other lanes: -1, 0). fp32 expf, denominator summed in k order (oracle: float64,
// |Δw| ≤ 1e-6). Everything stays in registers (K is a runtime value <= kMaxKS).
constexpr int kZJ = AMOE_MAX_E / kWarp;
__device__ __forceinline__ void route_load(const float* __restrict__ z, int E, int lane, float (&v)[kZJ]) {
#pragma unroll
  for (int j = 0; j < kZJ; ++j) {
    const int e = lane + kWarp * j;
    v[j] = e < E ? z[e] : -INFINITY;
  }
}
__device__ __forceinline__ void route_select(const float (&v)[kZJ], int E, int K, int lane, int& my_e, float& my_w) {
  uint32_t chosen = 0;
  float my_z = 0.f, z0 = 0.f;
  my_e = -1;
#pragma unroll 1
  for (int k = 0; k < K; ++k) {
    float bv = -INFINITY;
    int be = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < kZJ; ++j) {
      const int e = lane + kWarp * j;
      if (e < E && !((chosen >> j) & 1u) && (v[j] > bv || be == 0x7fffffff)) { bv = v[j]; be = e; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
    }
    if (k == 0) z0 = bv;
    if (lane == k) { my_e = be; my_z = bv; }
    if ((be & (kWarp - 1)) == lane) chosen |= 1u << (be / kWarp);
  }
  const float ex = lane < K ? expf(my_z - z0) : 0.f;
  float sum = 0.f;
#pragma unroll 1
  for (int k = 0; k < K; ++k) sum += __shfl_sync(0xffffffffu, ex, k);
  my_w = lane < K ? ex / sum : 0.f;
}

// Router gate: z[e] = Σ_j x[j]·wg[e][j] (+ bias[e]) for the token row x
// (storage T, already stored by this warp), fp32 accumulation (per lane over its 16-B chunks in
// column order, then the xor-tree warp sum). The row stays in registers (<= 16 chunks per lane);
// lane e % 32 receives z[e] in v[e / 32], the layout route_select expects.
template <typename T>
__device__ __noinline__ void gate_logits(const DevCtx& c, const T* __restrict__ x, const T* __restrict__ wg,
                                            const float* __restrict__ bias, int lane, float (&v)[kZJ]) {
  using V = Vec<T>;
  constexpr int MAXC = 16;
  uint4 xr[MAXC];
#pragma unroll
  for (int i = 0; i < MAXC; ++i) {
    const int col = (i * kWarp + lane) * V::N;
    if (col < c.d) xr[i] = *reinterpret_cast<const uint4*>(x + col);
  }
#pragma unroll
  for (int j = 0; j < kZJ; ++j) v[j] = -INFINITY;
#pragma unroll 1
  for (int e = 0; e < c.E; ++e) {
    const T* w = wg + (uint64_t)e * c.d;
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      const int col = (i * kWarp + lane) * V::N;
      if (col < c.d) {
        float xf[V::N], wf[V::N];
        V::unpack(xr[i], xf);
        V::unpack(*reinterpret_cast<const uint4*>(w + col), wf);
#pragma unroll
        for (int q = 0; q < V::N; ++q) acc = fmaf(xf[q], wf[q], acc);
      }
    }
    acc = warp_sum(acc);
    if (bias) acc += bias[e];
#pragma unroll
    for (int j = 0; j < kZJ; ++j)
      if (e == j * kWarp + lane) v[j] = acc;
  }
}

// The gate of `layer`, or (nullptr, nullptr) when the layer routes from the table.
__device__ __forceinline__ const uint64_t* gate_entry(const DevCtx& c, int layer) {
  return wsp<uint64_t>(c, c.rank, c.lay.gate) + 2 * (uint64_t)layer;
}

// ---------------------------------------------------------------------------- scatter (a2)
// Every thread of the CTA calls this. Legs with r >= 0 are appended to ring (r, q): one
// reservation atomic per (warp, queue) (__match_any_sync aggregation), entries written with
// the publication seq last, then one release-add of the commit counter per (warp, queue).
// Remote rings use system-scope atomics over NVLink.
__device__ void scatter_legs(const DevCtx& c, const PendingLeg* legs, int n) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool active = i < n && legs[i].r >= 0;
    const int r = active ? legs[i].r : 0;
    const int q = active ? legs[i].q : 0;
    const int key = active ? (r << 24 | q) : -1;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    // with peers, every producer of a ring (local or remote) uses system scope so that all
    // release/acquire pairs on the shared counters are morally strong
    const bool sys = c.G > 1;
    uint32_t pos0 = 0;
    if (active && lane == leader) {
      uint32_t* ctr = qctr_ptr(c, r, q);
      pos0 = atom_add_relaxed(ctr, (uint32_t)__popc(peers), sys);
      if (r == c.rank) {
        uint32_t head = ld_relaxed(ctr + 2);
        if (pos0 + (uint32_t)__popc(peers) - head > c.ring_cap) raise_fault(c, F_RING_OVERFLOW, q, pos0, head);
      }
    }
    pos0 = __shfl_sync(0xffffffffu, pos0, leader);
    if (active) {
      const uint32_t pos = pos0 + __popc(peers & ((1u << lane) - 1u));
      write_leg(ring_ptr(c, r, q), c.ring_mask, pos, legs[i].g, sys);
    }
    __syncwarp();
    if (active && lane == leader) {
      fence_sc(sys);
      red_add_release(qctr_ptr(c, r, q) + 1, (uint32_t)__popc(peers), sys);
    }
  }
}

// Fill the K (+S) legs of one routed token (lanes < K+S write their own leg).
__device__ __forceinline__ void make_legs(const DevCtx& c, int layer, int slot, int my_e, float my_w, int lane,
                                          PendingLeg* out) {
  if (lane < c.K) {
    PendingLeg p;
    if (my_e < 0 || my_e >= c.E) {
      raise_fault(c, F_EXPERT_RANGE, slot, my_e, layer);
      p.r = -1;
    } else {
      p.r = c.owner[my_e];
      p.q = layer * c.H + c.lq[my_e];
    }
    p.g.token_slot = slot; p.g.k = (int16_t)lane; p.g.home = (int16_t)c.rank; p.g.w = my_w; p.g.seq = 0;
    out[lane] = p;
  } else if (lane < c.KS) {
    PendingLeg p;
    p.r = c.rank;
    p.q = layer * c.H + c.Hr + (lane - c.K);
    p.g.token_slot = slot; p.g.k = (int16_t)lane; p.g.home = (int16_t)c.rank; p.g.w = 1.0f; p.g.seq = 0;
    out[lane] = p;
  }
}

// ---------------------------------------------------------------------------- RMSNorm (c7)
// x = store(h / sqrt(mean(h^2) + eps)) for one row held at `h` (storage T), warp-cooperative.
// The row was just stored by these lanes; it is re-read RB 16-B chunks per lane at a time, all
// loads of a batch before its stores (h and x may alias as far as the compiler knows, so a
// load-store loop would pay one L2 round trip per chunk: d / 256 of them per token).
template <typename T, int RB = 4>
__device__ __forceinline__ void rmsnorm_row(const DevCtx& c, const T* h, T* x, float ss, int lane) {
  using V = Vec<T>;
  constexpr int STEP = kWarp * V::N;
  const float r = 1.0f / sqrtf(ss / (float)c.d + c.eps);
  for (int col0 = lane * V::N; col0 < c.d; col0 += RB * STEP) {
    uint4 raw[RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int col = col0 + u * STEP;
      if (col < c.d) raw[u] = *reinterpret_cast<const uint4*>(h + col);
    }
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int col = col0 + u * STEP;
      if (col < c.d) {
        float f[V::N];
        V::unpack(raw[u], f);
#pragma unroll
        for (int j = 0; j < V::N; ++j) f[j] = f[j] * r;
        V::store(x + col, f);
      }
    }
  }
}

// ---------------------------------------------------------------------------- token_init

template <typename T>
__global__ void __launch_bounds__(kTokThreads) token_init_kernel(DevCtx c, const int32_t* __restrict__ slots,
                                                                 int n, const T* __restrict__ h0, int pass) {
  AMOE_PDL_ENTRY();
  using V = Vec<T>;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < n; i += nw) {
    const int slot = slots[i];
    if (slot < 0 || slot >= c.T) { if (lane == 0) raise_fault(c, F_SLOT_RANGE, slot, c.T, 0); continue; }
    T* h = wsp<T>(c, c.rank, c.lay.h) + (uint64_t)slot * c.d;
    T* x = wsp<T>(c, c.rank, c.lay.x) + (uint64_t)slot * c.d;
    const T* src = h0 + (uint64_t)i * c.d;
    float ss = 0.f;
    for (int col = lane * V::N; col < c.d; col += kWarp * V::N) {
      float f[V::N];
      V::load(src + col, f);
      V::store(h + col, f);
#pragma unroll
      for (int j = 0; j < V::N; ++j) ss += f[j] * f[j];
    }
    ss = warp_sum(ss);
    rmsnorm_row<T>(c, h, x, ss, lane);
    if (lane == 0) {
      unsigned long long* tt = wsp<unsigned long long>(c, c.rank, c.lay.tok_time) + 2 * (uint64_t)slot;
      tt[0] = globaltimer_ns();
      tt[1] = 0;
      wsp<int32_t>(c, c.rank, c.lay.tok_layer)[slot] = 0;
      wsp<int32_t>(c, c.rank, c.lay.tok_pass)[slot] = pass;
      wsp<uint32_t>(c, c.rank, c.lay.legs_done)[slot] = 0;
    }
  }
}

// ---------------------------------------------------------------------------- enqueue

__global__ void __launch_bounds__(kTokThreads) enqueue_kernel(DevCtx c, int layer, const int32_t* __restrict__ slots,
                                                              int n, const float* __restrict__ logits,
                                                              const int32_t* __restrict__ tidx,
                                                              const float* __restrict__ tw) {
  AMOE_PDL_ENTRY();
  __shared__ PendingLeg legs[kTPC * kMaxKS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // tokens per CTA chunk: a full chunk (kTPC) when there are enough tokens, otherwise spread so
  // every warp of the grid takes at most one token (few tokens: one latency chain, not kTPW)
  const int tpc = chunk_tokens(n);
  for (int base = blockIdx.x * tpc; base < n; base += gridDim.x * tpc) {
    for (int t = 0; t < kTPW; ++t) {
      const int lt = t * kTokWarps + warp;
      const int i = base + lt;
      PendingLeg* my = legs + lt * c.KS;
      if (lane < c.KS) my[lane].r = -1;
      if (lt >= tpc || i >= n) continue;
      const int slot = slots[i];
      if (slot < 0 || slot >= c.T) { if (lane == 0) raise_fault(c, F_SLOT_RANGE, slot, c.T, 1); continue; }
      int my_e = -1;
      float my_w = 0.f;
      if (logits) {
        float zv[kZJ];
        route_load(logits + (uint64_t)i * c.E, c.E, lane, zv);
        route_select(zv, c.E, c.K, lane, my_e, my_w);
      } else if (!tidx) {
        // gate routing on the token's x (amoe_set_gate); no gate for this layer is a fault
        const uint64_t* ge = gate_entry(c, layer);
        if (!ge[0]) { if (lane == 0) raise_fault(c, F_NO_ROUTER, slot, layer, 0); continue; }
        float zv[kZJ];
        if (c.dtype == AMOE_BF16)
          gate_logits<__nv_bfloat16>(c, wsp<__nv_bfloat16>(c, c.rank, c.lay.x) + (uint64_t)slot * c.d,
                                     reinterpret_cast<const __nv_bfloat16*>(ge[0]),
                                     reinterpret_cast<const float*>(ge[1]), lane, zv);
        else
          gate_logits<float>(c, wsp<float>(c, c.rank, c.lay.x) + (uint64_t)slot * c.d,
                             reinterpret_cast<const float*>(ge[0]), reinterpret_cast<const float*>(ge[1]), lane, zv);
        route_select(zv, c.E, c.K, lane, my_e, my_w);
      } else if (lane < c.K) {
        my_e = tidx[(uint64_t)i * c.K + lane];
        my_w = tw[(uint64_t)i * c.K + lane];
      }
      if (lane < c.K) {
        wsp<int32_t>(c, c.rank, c.lay.tok_idx)[(uint64_t)slot * c.K + lane] = my_e;
        wsp<float>(c, c.rank, c.lay.tok_w)[(uint64_t)slot * c.K + lane] = my_w;
      }
      if (lane == 0) {
        wsp<uint32_t>(c, c.rank, c.lay.legs_done)[slot] = 0;
        wsp<int32_t>(c, c.rank, c.lay.tok_layer)[slot] = layer;
      }
      make_legs(c, layer, slot, my_e, my_w, lane, my);
    }
    __syncthreads();
    scatter_legs(c, legs, kTPC * c.KS);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------- combine ring drain
// Single warp: n = published (commit) - head; commits are only ever observed after the entry
// writes (release/acquire), and when commit != reserve (a producer mid-flight on a peer) the
// published prefix is found by scanning the per-entry seq flags.
__global__ void cdrain_kernel(DevCtx c) {
  AMOE_PDL_ENTRY();
  uint32_t* ctr = wsp<uint32_t>(c, c.rank, c.lay.cctr);
  amoe_leg* ring = wsp<amoe_leg>(c, c.rank, c.lay.cring);
  int32_t* info = wsp<int32_t>(c, c.rank, c.lay.cinfo);
  const int lane = threadIdx.x;
  uint32_t head = ctr[2];
  uint32_t n;
  uint32_t cm = ld_acquire(ctr + 1);
  uint32_t rv = ld_relaxed(ctr + 0);
  if (cm == rv) {
    n = cm - head;
  } else {
    n = 0;
    for (;;) {
      const uint32_t pos = head + n + lane;
      const bool ok = (pos - head) < (rv - head) && ld_acquire(&ring[pos & c.cring_mask].seq) == pos + 1u;
      const uint32_t bad = __ballot_sync(0xffffffffu, !ok);
      if (bad) { n += __ffs(bad) - 1; break; }
      n += 32;
    }
  }
  if (n > c.cring_cap) { if (lane == 0) raise_fault(c, F_CRING_OVERFLOW, rv, head, 0); n = 0; }
  if (lane == 0) {
    info[0] = (int32_t)n;
    info[1] = (int32_t)head;
    ctr[2] = head + n;
  }
}

// ---------------------------------------------------------------------------- combine (a8)

// Router gate of a whole chunk on the tensor cores (bf16, every pending token at the same next
// layer): logits[32][E] = X[32 tokens, d] · Wgᵀ + b with warp-level mma.sync m16n8k16 (bf16 in,
// fp32 accumulate), fragments loaded straight from the x rows and Wg rows (L2 / L1). Tiles
// (m16 block, n8 block) go to the warps round-robin; rows of tokens without a gate read row 0.
__device__ __noinline__ void gate_chunk_mma(const DevCtx& c, const __nv_bfloat16* __restrict__ xbase,
                                               const int* s_slot, const __nv_bfloat16* __restrict__ wg,
                                               const float* __restrict__ bias, float* s_z, int zld, int warp,
                                               int lane) {
  const int ntiles = 2 * (c.E / 8);
  const int g = lane >> 2, q = lane & 3;
  for (int tile = warp; tile < ntiles; tile += kTokWarps) {
    const int mb = tile & 1, nt = tile >> 1;
    const int s0 = s_slot[mb * 16 + g], s1 = s_slot[mb * 16 + g + 8];
    const __nv_bfloat16* x0 = xbase + (uint64_t)(s0 < 0 ? 0 : s0) * c.d + 2 * q;
    const __nv_bfloat16* x1 = xbase + (uint64_t)(s1 < 0 ? 0 : s1) * c.d + 2 * q;
    const __nv_bfloat16* wr = wg + (uint64_t)(nt * 8 + g) * c.d + 2 * q;
    float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll 4
    for (int k0 = 0; k0 < c.d; k0 += 16) {
      const uint32_t a0 = *reinterpret_cast<const uint32_t*>(x0 + k0);
      const uint32_t a1 = *reinterpret_cast<const uint32_t*>(x1 + k0);
      const uint32_t a2 = *reinterpret_cast<const uint32_t*>(x0 + k0 + 8);
      const uint32_t a3 = *reinterpret_cast<const uint32_t*>(x1 + k0 + 8);
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(wr + k0);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(wr + k0 + 8);
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
          "{%0, %1, %2, %3};"
          : "+f"(d0), "+f"(d1), "+f"(d2), "+f"(d3)
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    const int col = nt * 8 + 2 * q;
    const float b0v = bias ? bias[col] : 0.f, b1v = bias ? bias[col + 1] : 0.f;
    float* z0 = s_z + (mb * 16 + g) * zld;
    float* z1 = s_z + (mb * 16 + g + 8) * zld;
    z0[col] = d0 + b0v; z0[col + 1] = d1 + b1v;
    z1[col] = d2 + b0v; z1[col + 1] = d3 + b1v;
  }
}

// KSM: compile-time bound on K+S (2, 4, 8 or 12) sizing the per-chunk leg registers.
template <typename T, int KSM, bool GATE>
__global__ void __launch_bounds__(kTokThreads, (KSM <= 4 && !GATE ? 4 : 2)) combine_kernel(DevCtx c, int retire_pass) {
  AMOE_PDL_ENTRY();
  using V = Vec<T>;
  __shared__ PendingLeg legs[kTPC * kMaxKS];
  __shared__ unsigned long long s_merged, s_retired;
  // GATE (bf16): tokens whose next layer routes with a gate are routed after the chunk's merges,
  // their logits computed for the whole chunk at once on the tensor cores
  constexpr int kZLD = GATE ? AMOE_MAX_E + 1 : 1;
  __shared__ float s_z[GATE ? kTPC * kZLD : 1];
  __shared__ int s_gslot[GATE ? kTPC : 1], s_glayer[GATE ? kTPC : 1], s_gpass[GATE ? kTPC : 1];
  __shared__ int s_guni;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* info = wsp<int32_t>(c, c.rank, c.lay.cinfo);
  uint32_t* cctr = wsp<uint32_t>(c, c.rank, c.lay.cctr);
  // G = 1: every entry of the combine ring was appended by this rank's earlier kernels (stream
  // order), so each CTA reads the published prefix [head, commit) itself and the last CTA to
  // finish advances the head (no cdrain launch); G > 1: cdrain_kernel's snapshot (peers may be
  // appending concurrently)
  int n;
  uint32_t start;
  if (c.G == 1) {
    start = cctr[2];
    n = (int)(ld_acquire(cctr + 1) - start);
    if ((uint32_t)n > c.cring_cap) {
      if (blockIdx.x == 0 && threadIdx.x == 0) raise_fault(c, F_CRING_OVERFLOW, cctr[0], start, 0);
      n = 0;
    }
  } else {
    n = info[0];
    start = (uint32_t)info[1];
  }
  const amoe_leg* ring = wsp<amoe_leg>(c, c.rank, c.lay.cring);
  T* hbase = wsp<T>(c, c.rank, c.lay.h);
  T* xbase = wsp<T>(c, c.rank, c.lay.x);
  const T* pool = wsp<T>(c, c.rank, c.lay.pool);
  const float* tokw = wsp<float>(c, c.rank, c.lay.tok_w);
  int32_t* tlayer = wsp<int32_t>(c, c.rank, c.lay.tok_layer);
  int32_t* tpass = wsp<int32_t>(c, c.rank, c.lay.tok_pass);
  if (threadIdx.x == 0) { s_merged = 0; s_retired = 0; }
  __syncthreads();
  const bool gate_tc = GATE && c.dtype == AMOE_BF16 && (c.E % 8) == 0;
  const int tpc = chunk_tokens(n);
  for (int base = blockIdx.x * tpc; base < n; base += gridDim.x * tpc) {
    for (int t = 0; t < kTPW; ++t) {
      const int lt = t * kTokWarps + warp;
      const int i = base + lt;
      PendingLeg* my = legs + lt * c.KS;
      if (lane < c.KS) my[lane].r = -1;
      if (GATE && lane == 0) s_gslot[lt] = -1;
      if (lt >= tpc || i >= n) continue;
      const uint32_t pos = start + (uint32_t)i;
      const amoe_leg e = ring[pos & c.cring_mask];
      if (e.seq != pos + 1u) { if (lane == 0) raise_fault(c, F_STALE_ENTRY, 0xffffffffu, pos, e.seq); continue; }
      const int slot = e.token_slot;
      // the token's next position (layer + 1, or layer 0 of the next pass) and, unless it
      // retires, its router logits there: loaded before the merge so their latency overlaps it
      int layer = tlayer[slot] + 1;
      int pass = tpass[slot];
      if (layer == c.L) { layer = 0; ++pass; }
      const bool retire = pass >= retire_pass;
      float zv[kZJ];
      const T* gw = nullptr;
      const float* gb = nullptr;
      if (GATE && !retire) {
        const uint64_t* ge = gate_entry(c, layer);
        gw = reinterpret_cast<const T*>(ge[0]);
        gb = reinterpret_cast<const float*>(ge[1]);
      }
      if (!retire && c.router && !gw)
        route_load(c.router + (((uint64_t)(pass % c.n_tab) * c.L + layer) * c.T + slot) * c.E, c.E, lane, zv);
      // h_new = store(h + Σ_k w_k O_k + Σ_j O_shared_j), ascending k then j, no FMA (c9);
      // shared legs use w = 1 (1·O == O exactly)
      float w[KSM];
#pragma unroll
      for (int k = 0; k < KSM; ++k) w[k] = k < c.K ? tokw[(uint64_t)slot * c.K + k] : 1.0f;
      T* h = hbase + (uint64_t)slot * c.d;
      const T* legrow = pool + (uint64_t)slot * c.KS * c.d;
      float ss = 0.f;
      for (int col = lane * V::N; col < c.d; col += kWarp * V::N) {
        // all K+S legs of this 16-byte chunk are loaded before the (ordered) accumulation, so
        // each lane keeps K+S+1 loads in flight (the leg count is a runtime value <= KSM)
        uint4 raw[KSM];
        const uint4 hraw = *reinterpret_cast<const uint4*>(h + col);
#pragma unroll
        for (int k = 0; k < KSM; ++k)
          if (k < c.KS) raw[k] = *reinterpret_cast<const uint4*>(legrow + (uint64_t)k * c.d + col);
        float acc[V::N];
        V::unpack(hraw, acc);
#pragma unroll
        for (int k = 0; k < KSM; ++k) {
          if (k < c.KS) {
            float o[V::N];
            V::unpack(raw[k], o);
            const float wk = w[k];
#pragma unroll
            for (int j = 0; j < V::N; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(wk, o[j]));
          }
        }
        V::store(h + col, acc);
#pragma unroll
        for (int j = 0; j < V::N; ++j) { const float r = V::round(acc[j]); ss += r * r; }
      }
      ss = warp_sum(ss);
      rmsnorm_row<T, (KSM >= 8 ? 4 : 2)>(c, h, xbase + (uint64_t)slot * c.d, ss, lane);
      if (lane == 0) { tlayer[slot] = layer; tpass[slot] = pass; atomicAdd(&s_merged, 1ull); }
      if (retire) {
        if (lane == 0) {
          atomicAdd(&s_retired, 1ull);
          wsp<unsigned long long>(c, c.rank, c.lay.tok_time)[2 * (uint64_t)slot + 1] = globaltimer_ns();
        }
        continue;
      }
      if (GATE && gw && gate_tc) {
        // routed after the chunk's merges (tensor-core gate over the chunk)
        if (lane == 0) { s_gslot[lt] = slot; s_glayer[lt] = layer; s_gpass[lt] = pass; }
        continue;
      }
      if (GATE && gw) {
        // the next layer's gate on the row just normalised (this warp stored x; same lanes)
        gate_logits<T>(c, xbase + (uint64_t)slot * c.d, gw, gb, lane, zv);
      } else if (!c.router) {
        if (lane == 0) raise_fault(c, F_NO_ROUTER, slot, layer, pass);
        continue;
      }
      int my_e;
      float my_w;
      route_select(zv, c.E, c.K, lane, my_e, my_w);
      if (lane < c.K) {
        wsp<int32_t>(c, c.rank, c.lay.tok_idx)[(uint64_t)slot * c.K + lane] = my_e;
        wsp<float>(c, c.rank, c.lay.tok_w)[(uint64_t)slot * c.K + lane] = my_w;
      }
      if (lane == 0) wsp<uint32_t>(c, c.rank, c.lay.legs_done)[slot] = 0;
      make_legs(c, layer, slot, my_e, my_w, lane, my);
    }
    if (gate_tc) {
      __syncthreads();                    // x rows of the chunk stored, gate list complete
      if (threadIdx.x == 0) {
        int u = -2;                       // -2: none pending, -1: mixed layers, else the layer
        for (int j = 0; j < kTPC; ++j)
          if (s_gslot[j] >= 0) u = (u == -2 || u == s_glayer[j]) ? s_glayer[j] : -1;
        s_guni = u;
      }
      __syncthreads();
      const int u = s_guni;
      if (u >= 0) {
        const uint64_t* ge = gate_entry(c, u);
        gate_chunk_mma(c, reinterpret_cast<const __nv_bfloat16*>(xbase), s_gslot,
                       reinterpret_cast<const __nv_bfloat16*>(ge[0]), reinterpret_cast<const float*>(ge[1]),
                       s_z, kZLD, warp, lane);
      }
      __syncthreads();
      if (u != -2) {
        for (int t = 0; t < kTPW; ++t) {
          const int lt = t * kTokWarps + warp;
          const int slot = s_gslot[lt];
          if (slot < 0) continue;
          const int layer = s_glayer[lt], pass = s_gpass[lt];
          float zv[kZJ];
          if (u >= 0) {
#pragma unroll
            for (int j = 0; j < kZJ; ++j) {
              const int e = lane + kWarp * j;
              zv[j] = e < c.E ? s_z[lt * kZLD + e] : -INFINITY;
            }
          } else {                        // mixed layers in the chunk: per-token gate
            const uint64_t* ge = gate_entry(c, layer);
            gate_logits<T>(c, xbase + (uint64_t)slot * c.d, reinterpret_cast<const T*>(ge[0]),
                           reinterpret_cast<const float*>(ge[1]), lane, zv);
          }
          int my_e;
          float my_w;
          route_select(zv, c.E, c.K, lane, my_e, my_w);
          if (lane < c.K) {
            wsp<int32_t>(c, c.rank, c.lay.tok_idx)[(uint64_t)slot * c.K + lane] = my_e;
            wsp<float>(c, c.rank, c.lay.tok_w)[(uint64_t)slot * c.K + lane] = my_w;
          }
          if (lane == 0) wsp<uint32_t>(c, c.rank, c.lay.legs_done)[slot] = 0;
          make_legs(c, layer, slot, my_e, my_w, lane, legs + lt * c.KS);
        }
      }
    }
    __syncthreads();
    scatter_legs(c, legs, kTPC * c.KS);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    unsigned long long* st = wsp<unsigned long long>(c, c.rank, c.lay.stats);
    if (s_merged) atomicAdd(st + 0, s_merged);
    if (s_retired) atomicAdd(st + 1, s_retired);
    if (c.G == 1) {
      // every CTA has read the head: the last one out consumes the prefix (info[2]: exit count)
      __threadfence();
      if (atomicAdd(reinterpret_cast<uint32_t*>(info + 2), 1u) == gridDim.x - 1) {
        cctr[2] = start + (uint32_t)n;
        info[2] = 0;
        __threadfence();
      }
    }
  }
}

// ---------------------------------------------------------------------------- direct merge (f3)
// Top-1 direct forwarding (with one expert per token there
// is no top-K merge to wait for, L227-L228: a token that is ready by itself skips the token
// pool). With K = 1 and no shared experts the rank that executed a token's leg merges it
// itself, right after the FFN: h ← store(h + w·O) (the combine's arithmetic, no FMA), x =
// RMSNorm(h) written back to the token's home, the next layer routed and the new leg scattered
// straight into the next expert's queue — no pool row, no leg counter, no combine ring, no merge
// launch on the home. The FFN output rows are this rank's group `out` rows; h, x and the token
// state stay on the home (NVLink peer loads/stores when remote). Routing: the router gate of
// the next layer (any G), or the router table (G = 1: the table is this rank's).
template <typename T, bool GATE>
__global__ void __launch_bounds__(kTokThreads) direct_merge_kernel(DevCtx c, GroupDev g, int retire_pass) {
  AMOE_PDL_ENTRY();
  using V = Vec<T>;
  __shared__ PendingLeg legs[kTPC * kMaxKS];
  __shared__ int pre[AMOE_MAX_GROUP + 1];
  __shared__ unsigned long long s_legs, s_remote;
  __shared__ int s_home[kTPC];                 // home of the token merged at chunk position lt (-1: none)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < g.nq; ++q) { pre[q] = acc; acc += g.qinfo[q]; }
    pre[g.nq] = acc;
    s_legs = 0; s_remote = 0;
  }
  __syncthreads();
  const int n = pre[g.nq];
  const bool sys = c.G > 1;
  const int tpc = chunk_tokens(n);
  for (int base = blockIdx.x * tpc; base < n; base += gridDim.x * tpc) {
    for (int t = 0; t < kTPW; ++t) {
      const int lt = t * kTokWarps + warp;
      const int i = base + lt;
      PendingLeg* my = legs + lt * c.KS;
      if (lane < c.KS) my[lane].r = -1;
      if (lane == 0) s_home[lt] = -1;
      if (lt >= tpc || i >= n) continue;
      int q = 0;
      while (q + 1 < g.nq && pre[q + 1] <= i) ++q;
      const int row = g.qinfo[AMOE_MAX_GROUP + q] + (i - pre[q]);
      const amoe_leg e = g.meta[row];
      const int home = e.home, slot = e.token_slot;
      if (home < 0 || home >= c.G || slot < 0 || slot >= c.T) {
        if (lane == 0) raise_fault(c, F_STALE_ENTRY, 0xfffffffeu, (uint32_t)row, e.seq);
        continue;
      }
      int32_t* tlayer = reinterpret_cast<int32_t*>(c.peer[home] + c.lay.tok_layer);
      int32_t* tpass = reinterpret_cast<int32_t*>(c.peer[home] + c.lay.tok_pass);
      int layer = tlayer[slot] + 1;
      int pass = tpass[slot];
      if (layer == c.L) { layer = 0; ++pass; }
      const bool retire = pass >= retire_pass;
      float zv[kZJ];
      const T* gw = nullptr;
      const float* gb = nullptr;
      if (GATE && !retire) {
        const uint64_t* ge = gate_entry(c, layer);
        gw = reinterpret_cast<const T*>(ge[0]);
        gb = reinterpret_cast<const float*>(ge[1]);
      }
      if (!retire && c.router && !gw)
        route_load(c.router + (((uint64_t)(pass % c.n_tab) * c.L + layer) * c.T + slot) * c.E, c.E, lane, zv);
      T* h = reinterpret_cast<T*>(c.peer[home] + c.lay.h) + (uint64_t)slot * c.d;
      T* x = reinterpret_cast<T*>(c.peer[home] + c.lay.x) + (uint64_t)slot * c.d;
      const T* orow = reinterpret_cast<const T*>(g.out) + (uint64_t)row * c.d;
      const float wk = e.w;
      float ss = 0.f;
      for (int col = lane * V::N; col < c.d; col += kWarp * V::N) {
        const uint4 hraw = *reinterpret_cast<const uint4*>(h + col);
        const uint4 oraw = *reinterpret_cast<const uint4*>(orow + col);
        float acc[V::N], o[V::N];
        V::unpack(hraw, acc);
        V::unpack(oraw, o);
#pragma unroll
        for (int j = 0; j < V::N; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(wk, o[j]));
        V::store(h + col, acc);
#pragma unroll
        for (int j = 0; j < V::N; ++j) { const float r = V::round(acc[j]); ss += r * r; }
      }
      ss = warp_sum(ss);
      rmsnorm_row<T>(c, h, x, ss, lane);
      if (lane == 0) {
        tlayer[slot] = layer;
        tpass[slot] = pass;
        atomicAdd(&s_legs, 1ull);
        if (home != c.rank) atomicAdd(&s_remote, 1ull);
        s_home[lt] = retire ? -2 - home : home;  // counted on the home after the chunk's scatter
      }
      if (retire) {
        if (lane == 0)
          reinterpret_cast<unsigned long long*>(c.peer[home] + c.lay.tok_time)[2 * (uint64_t)slot + 1] = globaltimer_ns();
        continue;
      }
      if (GATE && gw) {
        gate_logits<T>(c, x, gw, gb, lane, zv);
      } else if (!c.router) {
        if (lane == 0) raise_fault(c, F_NO_ROUTER, slot, layer, pass);
        continue;
      }
      int my_e;
      float my_w;
      route_select(zv, c.E, c.K, lane, my_e, my_w);
      if (lane < c.K) {
        reinterpret_cast<int32_t*>(c.peer[home] + c.lay.tok_idx)[(uint64_t)slot * c.K + lane] = my_e;
        reinterpret_cast<float*>(c.peer[home] + c.lay.tok_w)[(uint64_t)slot * c.K + lane] = my_w;
      }
      if (lane == 0) {
        PendingLeg p;
        if (my_e < 0 || my_e >= c.E) {
          raise_fault(c, F_EXPERT_RANGE, slot, my_e, layer);
          p.r = -1;
        } else {
          p.r = c.owner[my_e];
          p.q = layer * c.H + c.lq[my_e];
        }
        p.g.token_slot = slot; p.g.k = 0; p.g.home = (int16_t)home; p.g.w = my_w; p.g.seq = 0;
        my[0] = p;
      }
    }
    __syncthreads();
    scatter_legs(c, legs, kTPC * c.KS);
    __syncthreads();
    // merged (and retired) counts on each token's home, once its state and next leg are
    // visible: the home's amoe_run reads them for quiescence, as it reads the combine's
    if (threadIdx.x < kTPC && s_home[threadIdx.x] != -1) {
      const int v = s_home[threadIdx.x];
      const int home = v >= 0 ? v : -2 - v;
      unsigned long long* hst = reinterpret_cast<unsigned long long*>(c.peer[home] + c.lay.stats);
      fence_sc(sys);
      if (sys) {
        atomicAdd_system(hst + 0, 1ull);
        if (v < 0) atomicAdd_system(hst + 1, 1ull);
      } else {
        atomicAdd(hst + 0, 1ull);
        if (v < 0) atomicAdd(hst + 1, 1ull);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    unsigned long long* st = wsp<unsigned long long>(c, c.rank, c.lay.stats);
    if (s_legs) atomicAdd(st + 2, s_legs);
    if (s_remote) atomicAdd(st + 3, s_remote);
  }
}

int launch_direct_merge(const DevCtx& c, const GroupDev& g, int retire_pass, int num_sms, cudaStream_t s) {
  const int grid = num_sms * 4;
  if (c.dtype == AMOE_BF16) {
    if (c.gate_on) launch_pdl(direct_merge_kernel<__nv_bfloat16, true>, dim3(grid), dim3(kTokThreads), 0, s, c, g, retire_pass);
    else launch_pdl(direct_merge_kernel<__nv_bfloat16, false>, dim3(grid), dim3(kTokThreads), 0, s, c, g, retire_pass);
  } else {
    if (c.gate_on) launch_pdl(direct_merge_kernel<float, true>, dim3(grid), dim3(kTokThreads), 0, s, c, g, retire_pass);
    else launch_pdl(direct_merge_kernel<float, false>, dim3(grid), dim3(kTokThreads), 0, s, c, g, retire_pass);
  }
  return 1;
}

// done[base + rank] = value on every rank (base 0: quiescence epoch; base AMOE_MAX_G: the
// AMOE_SYNC layer-barrier sequence). Release: the stores of this rank's earlier kernels are
// visible to a peer that observes the flag.
__global__ void announce_kernel(DevCtx c, uint32_t value, int base) {
  AMOE_PDL_ENTRY();
  const int r = threadIdx.x;
  if (r < c.G) st_release(wsp<uint32_t>(c, r, c.lay.done) + base + c.rank, value, r != c.rank);
}

// ---------------------------------------------------------------------------- launchers

int launch_token_init(const DevCtx& c, const int32_t* slots, int n, const void* h0, int pass, cudaStream_t s) {
  const int grid = (n + kTokWarps - 1) / kTokWarps < 1184 ? (n + kTokWarps - 1) / kTokWarps : 1184;
  if (n <= 0) return 0;
  if (c.dtype == AMOE_BF16)
    launch_pdl(token_init_kernel<__nv_bfloat16>, dim3(grid), dim3(kTokThreads), 0, s, c, slots, n, (const __nv_bfloat16*)h0, pass);
  else
    launch_pdl(token_init_kernel<float>, dim3(grid), dim3(kTokThreads), 0, s, c, slots, n, (const float*)h0, pass);
  return 1;
}

int launch_enqueue(const DevCtx& c, int layer, const int32_t* slots, int n, const float* logits,
                   const int32_t* tidx, const float* tw, cudaStream_t s) {
  if (n <= 0) return 0;
  int grid = (n + kTokWarps - 1) / kTokWarps;     // chunk_tokens: one token per warp when few
  if (grid > 1184) grid = 1184;
  launch_pdl(enqueue_kernel, dim3(grid), dim3(kTokThreads), 0, s, c, layer, slots, n, logits, tidx, tw);
  return 1;
}

template <typename T, int KSM, bool GATE>
static void launch_combine_t(const DevCtx& c, int retire_pass, int num_sms, cudaStream_t s) {
  // persistent grid: every resident CTA slot once (no tail wave), capped by the worst case (all
  // homed tokens ready); CTAs loop over 32-token chunks of the ready list. Occupancy is a
  // property of the kernel (same on every B200); the SM count is the context's (AMOE_NUM_SMS
  // partitions in the G-rank emulation)
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, combine_kernel<T, KSM, GATE>, kTokThreads, 0);
    if (occ < 1) occ = 1;
  }
  int grid = (c.T + kTPC - 1) / kTPC;
  if (grid > num_sms * occ) grid = num_sms * occ;
  launch_pdl(combine_kernel<T, KSM, GATE>, dim3(grid), dim3(kTokThreads), 0, s, c, retire_pass);
}

template <typename T, bool GATE>
static void launch_combine_g(const DevCtx& c, int retire_pass, int num_sms, cudaStream_t s) {
  const int ksm = c.KS <= 2 ? 2 : c.KS <= 4 ? 4 : c.KS <= 8 ? 8 : 12;
  if (ksm == 2) launch_combine_t<T, 2, GATE>(c, retire_pass, num_sms, s);
  else if (ksm == 4) launch_combine_t<T, 4, GATE>(c, retire_pass, num_sms, s);
  else if (ksm == 8) launch_combine_t<T, 8, GATE>(c, retire_pass, num_sms, s);
  else launch_combine_t<T, 12, GATE>(c, retire_pass, num_sms, s);
}

int launch_combine(const DevCtx& c, int retire_pass, int num_sms, cudaStream_t s) {
  if (c.G > 1) launch_pdl(cdrain_kernel, dim3(1), dim3(32), 0, s, c);   // G = 1: inside the combine
  if (c.dtype == AMOE_BF16) {
    if (c.gate_on) launch_combine_g<__nv_bfloat16, true>(c, retire_pass, num_sms, s);
    else launch_combine_g<__nv_bfloat16, false>(c, retire_pass, num_sms, s);
  } else {
    if (c.gate_on) launch_combine_g<float, true>(c, retire_pass, num_sms, s);
    else launch_combine_g<float, false>(c, retire_pass, num_sms, s);
  }
  return c.G > 1 ? 2 : 1;
}

int launch_announce(const DevCtx& c, uint32_t value, int base, cudaStream_t s) {
  launch_pdl(announce_kernel, dim3(1), dim3(32), 0, s, c, value, base);
  return 1;
}

}  // namespace amoe
