// amoe_internal.cuh — workspace layout, device context and memory-ordering helpers shared by
// the libamoe kernels (sm_100a). Not part of the C ABI (see include/amoe.h).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "amoe.h"

namespace amoe {

constexpr int kWarp = 32;
constexpr int kMaxKS = 12;          // K + S legs per token
constexpr int kRowAlign = 128;      // group rows are allocated per queue in multiples of this
constexpr int kSplitSlots = 512;    // split-K tile slots (counters)
constexpr int kSplitUnits = 2048;   // split-K partial tiles (128 x 256 fp32 each): 256 MB
constexpr int kColdCtr = 16384;     // cold-kernel flags and counters (u32), DESIGN.md §5.4

// Device fault codes latched into the error word.
enum Fault : uint32_t {
  F_NONE = 0,
  F_RING_OVERFLOW = 1,    // args: queue, reserve, head
  F_LEG_OVERCOUNT = 2,    // args: home slot, count, k
  F_EXPERT_RANGE = 3,     // args: slot, expert, layer
  F_NOT_HOSTED = 4,       // args: layer, expert, rank
  F_CRING_OVERFLOW = 5,   // args: reserve, head
  F_SLOT_RANGE = 6,       // args: slot, T
  F_STALE_ENTRY = 7,      // args: queue, position, seq
  F_NO_ROUTER = 8,        // args: slot, layer, pass (needs amoe_set_router or amoe_set_gate)
  F_PEER_ABORT = 9,       // args: peer rank whose fault (or timeout) aborted this rank's amoe_run (host-latched)
  F_RUN_TIMEOUT = 10,     // args: seconds, merged, expected (host-latched: AMOE_RUN_TIMEOUT expired, G > 1)
  F_LOST_LEG = 11,        // args: stranded token slot, its layer, leg columns returned (host-latched, G == 1)
  F_HEAD_MISMATCH = 12,   // args: queue, the drain's start position, the queue's consumer head (cold pick)
};
// done[] value a faulting rank stores into every peer: never equal to a run epoch
constexpr uint32_t kAbortEpoch = 0xFFFFFFFFu;

// Byte offsets of every object inside a rank's workspace. Identical on every rank (the
// layout depends only on the config), so a peer object's address is peer_base + offset.
struct Layout {
  uint64_t err;        // u32[8]: code, a0, a1, a2
  uint64_t stats;      // u64[8]: 0 merges, 1 retired, 2 legs executed, 3 legs sent remote
  uint64_t done;       // u32[AMOE_MAX_G]: done epoch per rank (written by that rank)
  uint64_t gtot;       // u32[L]: box-wide queued legs per block, every rank's queues (AMOE_DEFRAG_GLOBAL)
  uint64_t qctr;       // u32[L*H][4]: reserve, commit, head, pad
  uint64_t rings;      // amoe_leg[L*H][ring_cap]
  uint64_t cctr;       // u32[4]: combine ring reserve, commit, head, pad
  uint64_t cring;      // amoe_leg[cring_cap]
  uint64_t cinfo;      // i32[4]: combine drain n, start
  uint64_t sched;      // u32[4]: FFN die-aware tile claims {die 0, die 1, finished clusters, pad}
  uint64_t split_cnt;  // u32[kSplitSlots]: split-K arrival counters (self-resetting)
  uint64_t cold;       // u32[kColdCtr]: cold fused kernel: drain flag, gather arrivals, exits, partial flags, act counts
  uint64_t h, x;       // [T][d]
  uint64_t pool;       // [T][K+S][d]
  uint64_t legs_done;  // u32[T]
  uint64_t tok_layer;  // i32[T]
  uint64_t tok_pass;   // i32[T]
  uint64_t tok_w;      // f32[T][K]
  uint64_t tok_idx;    // i32[T][K]
  uint64_t tok_time;   // u64[T][2]: globaltimer (ns) at admission (token_init) and at retirement
  uint64_t wmaps;      // CUtensorMap[L*H][3]
  uint64_t cmaps;      // CUtensorMap[L*H][4]: K-block views (3-D) W1 x2, W3 x2, W2 x2, W2 x1 (cold kernel)
  uint64_t wptrs;      // u64[L*H][3]
  uint64_t gate;       // u64[L][2]: router gate weights [E][d] (storage dtype) and bias [E] fp32, or 0
  uint64_t s_tile, s_meta, s_qinfo, s_act, s_out;   // amoe_run's group scratch
  uint64_t split_part; // f32 split-K partials: kSplitUnits x 128 rows x 256 columns
  uint64_t total;
  int32_t rows_cap;
  int32_t pad_;
};

// Everything a kernel needs to address local and peer objects. Passed by value (param space).
struct DevCtx {
  int32_t L, E, K, S, d, ff, G, rank, T, dtype, H, Hr, KS, esize;
  uint32_t ring_cap, ring_mask, cring_cap, cring_mask;
  float eps;
  int32_t n_tab;
  const float* router;               // local [n_tab][L][T][E] or null
  int32_t gate_on;                   // some layer has a router gate (amoe_set_gate)
  uint32_t* xlog;                    // checked-mode execution log (amoe_set_exec_log) or null
  int32_t die_cnt[2];                // SMs on each die (die_probe); die_cnt[1] == 0: no die split
  int32_t pad_die;
  uint64_t die_mask[4];              // bit smid set: SM on die 1
  Layout lay;
  uint64_t peer[AMOE_MAX_G];         // workspace base per rank; peer[rank] = local
  int16_t lq[AMOE_MAX_E];            // local queue index of routed expert e on its owner
  uint8_t owner[AMOE_MAX_E];
};

// One grouped execution as the queue kernels see it.
struct GroupDev {
  int32_t nq;
  int32_t rows_cap;
  int32_t max_tokens;
  int32_t exact;                 // 1: drain exactly cap[q] legs per queue (the scheduler's count)
  int32_t cap[AMOE_MAX_GROUP];
  int32_t* qinfo;          // [3*AMOE_MAX_GROUP]: n, row_off, start
  amoe_leg* meta;
  void* tile;
  void* out;
  int32_t qid[AMOE_MAX_GROUP];   // local queue index l*H + lq
};

// Grouped FFN launch description (tensor-core path).
struct FfnLaunch {
  int nq;
  const int32_t* qinfo;
  const CUtensorMap* wmaps;      // device [L*H][3]
  int wslot[AMOE_MAX_GROUP];     // (l*H + lq) * 3
  int rows_hint;                 // amoe_group::max_rows_hint
  int exact_max_n = -1;          // amoe_run's pipelined picks: the largest queue's exact drain count
                                 // (-1: unknown); a launch whose largest queue spans >= 2 M tiles
                                 // never splits K, so its split-K reduction is not launched
};

template <typename T>
__device__ __forceinline__ T* wsp(const DevCtx& c, int r, uint64_t off) {
  return reinterpret_cast<T*>(c.peer[r] + off);
}

// ------------------------------------------------------------------ memory-ordering helpers
// Local objects use .gpu scope; objects on (or shared with) a peer GPU use .sys scope so the
// NVLink peer observes the ordering (PTX memory model, scopes).

__device__ __forceinline__ uint32_t atom_add_relaxed(uint32_t* p, uint32_t v, bool sys) {
  uint32_t old;
  if (sys) asm volatile("atom.relaxed.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  else     asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_acqrel(uint32_t* p, uint32_t v, bool sys) {
  uint32_t old;
  if (sys) asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  else     asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_add_release(uint32_t* p, uint32_t v, bool sys) {
  uint32_t old;
  if (sys) asm volatile("atom.release.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  else     asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(uint32_t* p, uint32_t v, bool sys) {
  if (sys) asm volatile("red.release.sys.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
  else     asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
  else     asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sc(bool sys) {
  if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else     asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Latch the first device fault (later faults keep the first one's arguments).
__device__ __forceinline__ void raise_fault(const DevCtx& c, uint32_t code, uint32_t a0, uint32_t a1,
                                            uint32_t a2) {
  uint32_t* e = wsp<uint32_t>(c, c.rank, c.lay.err);
  if (atomicCAS(e, 0u, code) == 0u) {
    e[1] = a0; e[2] = a1; e[3] = a2;
    __threadfence();
  }
}

// ------------------------------------------------------------------ checked-mode execution log
// (amoe_set_exec_log): header u32[8] {executions, legs, exec capacity, leg capacity}, then exec
// records u32[4] {qid, start, n, leg offset}, then the drained legs (amoe_leg, seq := pass).
constexpr int kXlogHeader = 8;
__device__ __forceinline__ uint32_t* xlog_exec(uint32_t* xl) { return xl + kXlogHeader; }
__device__ __forceinline__ amoe_leg* xlog_legs(uint32_t* xl) {
  return reinterpret_cast<amoe_leg*>(xl + kXlogHeader + 4 * (uint64_t)xl[2]);
}

// ------------------------------------------------------------------ µ-queue rings

__device__ __forceinline__ uint32_t* qctr_ptr(const DevCtx& c, int r, int q) {
  return wsp<uint32_t>(c, r, c.lay.qctr) + 4 * q;
}
__device__ __forceinline__ amoe_leg* ring_ptr(const DevCtx& c, int r, int q) {
  return wsp<amoe_leg>(c, r, c.lay.rings) + (uint64_t)q * c.ring_cap;
}

// Write one leg into slot `pos` of a ring (the seq field is the publication flag, last).
__device__ __forceinline__ void write_leg(amoe_leg* ring, uint32_t mask, uint32_t pos,
                                          const amoe_leg& g, bool sys) {
  amoe_leg* e = ring + (pos & mask);
  int2 a;
  a.x = g.token_slot;
  a.y = (int)((uint32_t)(uint16_t)g.k | ((uint32_t)(uint16_t)g.home << 16));
  *reinterpret_cast<int2*>(e) = a;
  e->w = g.w;
  st_release(&e->seq, pos + 1u, sys);
}

// ------------------------------------------------------------------ token pool (a7 -> a8)
// A leg's output row is returned in pieces (column ranges: the fused down-GEMM epilogues store
// one N tile, or one slice of a split tile, at a time), counted in columns; the token is
// complete when all (K+S) * d columns of its legs arrived.
__device__ __forceinline__ uint32_t pieces_per_token(const DevCtx& c) { return (uint32_t)c.KS * (uint32_t)c.d; }

// Count `pieces` returned columns of token `slot` on `home` (release: the caller's pool stores
// happen before); the arrival completing the token appends it to the home's combine ring.
__device__ __forceinline__ void leg_pieces_done(const DevCtx& c, int home, int slot, int k, uint32_t pieces) {
  const bool sys = c.G > 1;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(c.peer[home] + c.lay.legs_done) + slot;
  // release-only increment (an acq_rel RMW costs a MEMBAR + L1 invalidate per piece); only the
  // completing arrival needs the acquire side, which it takes with a fence before publishing
  const uint32_t old = atom_add_release(cnt, pieces, sys);
  const uint32_t total = pieces_per_token(c);
  if (old + pieces > total) raise_fault(c, F_LEG_OVERCOUNT, slot, old + pieces, k);
  if (old + pieces == total) {
    fence_sc(sys);
    uint32_t* cctr = reinterpret_cast<uint32_t*>(c.peer[home] + c.lay.cctr);
    amoe_leg* cring = reinterpret_cast<amoe_leg*>(c.peer[home] + c.lay.cring);
    const uint32_t pos = atom_add_relaxed(cctr, 1u, sys);
    amoe_leg t;
    t.token_slot = slot; t.k = 0; t.home = (int16_t)home; t.w = 0.f; t.seq = 0;
    write_leg(cring, c.cring_mask, pos, t, sys);
    red_add_release(cctr + 1, 1u, sys);
  }
}

// ------------------------------------------------------------------ storage-type vectors
// 16-byte vectors: 8 bf16 or 4 fp32 values.

template <typename T> struct Vec;
template <> struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void load(const __nv_bfloat16* p, float* f) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) { float2 t = __bfloat1622float2(b[i]); f[2 * i] = t.x; f[2 * i + 1] = t.y; }
  }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, const float* f) {
    uint4 u;
    __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
  // value as stored (rounded), for sums over stored values
  __device__ __forceinline__ static float round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
  __device__ __forceinline__ static void unpack(const uint4& u, float* f) {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) { float2 t = __bfloat1622float2(b[i]); f[2 * i] = t.x; f[2 * i + 1] = t.y; }
  }
};
template <> struct Vec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void load(const float* p, float* f) {
    float4 u = *reinterpret_cast<const float4*>(p);
    f[0] = u.x; f[1] = u.y; f[2] = u.z; f[3] = u.w;
  }
  __device__ __forceinline__ static void store(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  }
  __device__ __forceinline__ static float round(float v) { return v; }
  __device__ __forceinline__ static void unpack(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y); f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
  }
};

// ------------------------------------------------------------------ programmatic dependent launch
// Every libamoe kernel is launched with programmatic stream serialisation (launch_pdl): it may be
// scheduled while the previous kernel of the stream drains, runs AMOE_PDL_ENTRY first — wait
// until that kernel completed and its memory is visible, then let the next kernel be scheduled —
// so a kernel boundary costs no launch latency. (griddepcontrol.* are no-ops for normal launches.)
#define AMOE_PDL_ENTRY()                                                      \
  do {                                                                         \
    asm volatile("griddepcontrol.wait;" ::: "memory");                         \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");            \
  } while (0)

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Copy `bytes` (multiple of 16) with a warp, 16 B per lane, 4 loads in flight per lane.
__device__ __forceinline__ void warp_copy(void* dst, const void* src, int bytes, int lane) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  const int n = bytes >> 4;
  int i = lane;
  for (; i + 96 < n; i += 128) {
    uint4 a = s[i], b = s[i + 32], c2 = s[i + 64], e = s[i + 96];
    d[i] = a; d[i + 32] = b; d[i + 64] = c2; d[i + 96] = e;
  }
  for (; i < n; i += 32) d[i] = s[i];
}

}  // namespace amoe
