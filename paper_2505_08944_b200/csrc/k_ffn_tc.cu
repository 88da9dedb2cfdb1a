// k_ffn_tc.cu — a5/a6: grouped expert FFN on the 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel per GEMM of the SwiGLU expert
// (reading c1: O = W2 (silu(W1 x) ⊙ W3 x)), covering every queue of a grouped pick:
//   MODE_GATEUP: D[128 x 256] = X_tile[128 x d] · [W1 rows n0..n0+127 ; W3 rows n0..n0+127]ᵀ,
//                epilogue act = bf16(silu(D[:, :128]) ⊙ D[:, 128:])       (SwiGLU fused)
//   MODE_DOWN  : D[128 x BN] = act_tile[128 x ff] · W2[n0..n0+BN-1, :]ᵀ, epilogue out = bf16(D)
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = tcgen05.mma issuer (one thread),
// warp 2 = TMEM allocator, warps 4..7 = epilogue (TMEM -> registers -> global).
// Operands: TMA 2D tiles, 128-byte swizzle, K-major; 4-stage smem ring (48 KB/stage) with
// full/empty mbarriers; two 256-column fp32 accumulators in TMEM so the epilogue of tile i
// overlaps the main loop of tile i+1. Tiles of a queue are rasterised in groups of 16 M-tiles
// so concurrently running CTAs share the weight slab and the token rows through L2.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "amoe_internal.cuh"
#include "tc_ptx.cuh"

namespace amoe {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;              // 64 bf16 = 128 B = one swizzle atom row
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int B_BYTES = 256 * BK * 2;           // 32 KB (max BN = 256)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int THREADS = 256;
constexpr int GROUP_M = 16;
// default FFN variant: the CTA pair (UMMA M=256, cta_group::2) when d % 256 == 0 — measured
// 1.33 vs 1.27 TFLOP/s per W under the power cap (profiles/r01_ffn_power.md); AMOE_FFN_1CTA=1
// selects the 1-CTA kernel (UMMA M=128), which also serves d % 256 != 0
constexpr bool kDefault1Cta = false;
constexpr int TMEM_COLS = 512;
constexpr int EPI_STAGE_BYTES = 4 * 4096;       // epilogue store staging, 4 KB per epilogue warp
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 4096 + EPI_STAGE_BYTES + 1024;   // + barriers/tables + align

enum Mode { MODE_GATEUP = 0, MODE_DOWN = 1 };

struct FfnArgs {
  int32_t nq;
  int32_t n_tiles;       // N tiles per queue
  int32_t k_blocks;      // K / 64
  int32_t out_ld;        // output row stride (elements)
  int32_t out_cols;      // valid output columns
  int32_t w_which;       // 0 (W1; W3 = +1) or 2 (W2) within a queue's 3 tensor maps
  int32_t group_m;       // M tiles per raster group (L2 reuse of the weight slab)
  int32_t fuse;          // DOWN: 1 = store rows straight into the home token pools (fused a7)
  int32_t ring_legs;     // 1 = the drained legs are read from the µ-queue rings (no meta copy)
  int32_t gather;        // GATEUP: A rows gathered from x by token slot: 1 = TMA tile::gather4,
                         // 2 = cp.async by the producer warp (CTA-pair kernel only)
  int32_t allow_split;   // split K when the output tiles cannot fill the machine (cold experts)
  int32_t atrim;         // partial M tiles load only their valid A rows
  int32_t die_sched;     // CTA-pair kernels: 0 static raster; dynamic claims through the unit
                         // ring: 3 one list, 1 per-die N-tile shares (AMOE_FFN_SCHED)
  uint32_t* sched;       // u32[4] claim counters {die 0, die 1, finished clusters} (self-resetting)
  float* part;           // split-K fp32 partials (workspace)
  uint32_t* cnt;         // split-K per-slot arrival counters (workspace, self-resetting)
  const amoe_leg* meta;  // [rows] drained legs (fused forward) when !ring_legs
  const int32_t* qinfo;
  const CUtensorMap* wmaps;
  __nv_bfloat16* out;
  int32_t wslot[AMOE_MAX_GROUP];   // (l*H + lq) * 3
};

// ------------------------------------------------------------------ tile schedule
struct Sched {
  int nq, n_tiles, total, group;
  const int* n;
  const int* off;
  const int* pre;     // tile prefix per queue
  __device__ __forceinline__ void decode(int t, int& q, int& m, int& nb) const {
    int lo = 0, hi = nq - 1;
    while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (pre[mid] <= t) lo = mid; else hi = mid - 1; }
    q = lo;
    const int u = t - pre[q];
    const int m_tiles = (n[q] + BM - 1) / BM;
    const int gsz = group * n_tiles;
    const int g = u / gsz;
    const int first_m = g * group;
    const int gm = min(m_tiles - first_m, group);
    const int r = u - g * gsz;
    m = first_m + r % gm;
    nb = r / gm;
  }
};

// The epilogue warps (threads [first, first+128)) wait for an accumulator: one elected thread
// sleeps on the mbarrier, the others block on a hardware named barrier (no issue slots).
__device__ __forceinline__ void epi_wait(uint32_t bar, uint32_t parity, int tid, int first) {
  if (tid == first) mbar_wait(bar, parity);
  asm volatile("bar.sync 1, 128;" ::: "memory");
}
// ... and release it once every thread's TMEM loads completed: one arrive (count 1).
__device__ __forceinline__ void epi_release_local(uint32_t bar, int tid, int first) {
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (tid == first) mbar_arrive(bar);
}

// ------------------------------------------------------------------ fused a7 (forward)
// DOWN epilogue destination of a row: the group's `out` buffer, or — fused forward — the leg's
// slot in its home's token pool (local or NVLink peer store), pool[home][slot][k][:].
// The drained leg of row `row` of queue q: from the materialised meta rows, or (ring_legs) from
// the µ-queue ring itself — position start[q] + row — when the gather was fused into the A load.
__device__ __forceinline__ amoe_leg leg_of_row(const FfnArgs& a, const DevCtx& dc, int q, int row, int grow,
                                               const int* s_start) {
  if (a.ring_legs) {
    const amoe_leg* ring = reinterpret_cast<const amoe_leg*>(dc.peer[dc.rank] + dc.lay.rings) +
                           (uint64_t)(a.wslot[q] / 3) * dc.ring_cap;
    return ring[((uint32_t)s_start[q] + (uint32_t)row) & dc.ring_mask];
  }
  return a.meta[grow];
}
template <int MODE>
__device__ __forceinline__ __nv_bfloat16* down_row_dst(const FfnArgs& a, const DevCtx& dc, int q, int row, int grow,
                                                       const int* s_start, bool valid, amoe_leg& leg) {
  if (MODE == MODE_DOWN && a.fuse) {
    if (!valid) return nullptr;
    leg = leg_of_row(a, dc, q, row, grow, s_start);
    return reinterpret_cast<__nv_bfloat16*>(dc.peer[leg.home] + dc.lay.pool) +
           ((uint64_t)leg.token_slot * dc.KS + (uint64_t)leg.k) * dc.d;
  }
  return a.out + (uint64_t)grow * a.out_ld;
}
// ------------------------------------------------------------------ epilogue (shared by both kernels)
// One row per thread leaves TMEM (tcgen05.ld 32x32b: lane = accumulator row). Stored directly,
// every store instruction of a warp would touch 32 rows (32 half-filled sectors in 32 lines);
// instead each 64-column chunk of the warp's 32 rows goes through a 4 KB smem stage (16-B
// chunks XOR-swizzled by row: conflict-free both ways) and leaves as 4 whole 128-B row lines
// per instruction.
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
// w: this lane's row (NW packed bf16x2 words = 2·NW columns starting at column col0 of the row
// at dst; dst == nullptr: row not stored). ncols: valid columns of the row segment.
template <int NW>
__device__ __forceinline__ void store_rows_staged(const uint32_t (&w)[NW], __nv_bfloat16* dst, int col0, int ncols,
                                                  uint32_t stage, int lane) {
  static_assert(NW % 32 == 0, "64-column chunks");
  const int c = lane & 7;
  __nv_bfloat16* rdst[8];                 // destination rows 4 s + lane / 8 of this lane's stores
#pragma unroll
  for (int s = 0; s < 8; ++s)
    rdst[s] = reinterpret_cast<__nv_bfloat16*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), 4 * s + (lane >> 3)));
#pragma unroll
  for (int ch = 0; ch < NW / 32; ++ch) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      sts128(stage + lane * 128 + ((j ^ (lane & 7)) << 4), w[ch * 32 + 4 * j], w[ch * 32 + 4 * j + 1],
             w[ch * 32 + 4 * j + 2], w[ch * 32 + 4 * j + 3]);
    __syncwarp();
    const int col = ch * 64 + c * 8;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int r = 4 * s + (lane >> 3);
      const uint4 v = lds128(stage + r * 128 + ((c ^ (r & 7)) << 4));
      if (rdst[s] && col < ncols) *reinterpret_cast<uint4*>(rdst[s] + col0 + col) = v;
    }
    __syncwarp();
  }
}

// Fused forward (a7) leg counting, one unit behind the stores: the row's pieces of a tile are
// counted on the token's leg counter only at the next tile's epilogue (or at the kernel's end),
// after a fence that by then finds those stores long completed — so the epilogue never waits
// for its own output stores to drain (ncu: the per-tile fence was the down GEMM epilogue's top
// stall on DeepSeek-shaped layers).
struct PendCount {
  amoe_leg leg;
  int32_t pieces;   // 0: nothing pending for this lane's row
  int32_t nb;
};
__device__ __forceinline__ void flush_count(const DevCtx& dc, PendCount& pend, uint32_t (&fwd)[2]) {
  if (!__any_sync(0xffffffffu, pend.pieces > 0)) return;
  // every lane orders its own (staged) stores, then the row's owner lane counts the pieces
  fence_sc(dc.G > 1);
  __syncwarp();
  if (pend.pieces > 0) {
    leg_pieces_done(dc, pend.leg.home, pend.leg.token_slot, pend.leg.k, (uint32_t)pend.pieces);
    if (pend.nb == 0) { fwd[0] += 1; fwd[1] += (pend.leg.home != dc.rank); }
  }
  pend.pieces = 0;
}

// Non-split epilogue of one tile: every TMEM column this thread needs is loaded (and packed to
// bf16) first, the accumulator is released to the MMA issuer, and only then do the global
// stores (and, fused forward, the leg-piece counting) run — off the MMA's critical path.
// GATEUP: act = bf16(silu(g)·u), 128 columns; DOWN: out / home pool = bf16(v), BN columns.
#ifndef AMOE_EPI_LD
#define AMOE_EPI_LD 4
#endif
// TMEM loads per tcgen05.wait::ld in the epilogue (2 or 4): each wait is a full TMEM round trip.
constexpr int EPI_LD = AMOE_EPI_LD;

template <int MODE, int BN, typename Release>
__device__ __forceinline__ void epilogue_tile(const FfnArgs& args, const DevCtx& dc, uint32_t taddr, bool valid,
                                              __nv_bfloat16* orow, int nb, const amoe_leg& leg, uint32_t stage,
                                              int lane, uint32_t (&fwd)[2], PendCount& pend, Release release) {
  constexpr int NW = (MODE == MODE_GATEUP) ? 64 : BN / 2;
  uint32_t w[NW];
  if (MODE == MODE_GATEUP) {
#pragma unroll
    for (int ch = 0; ch < 8; ch += EPI_LD / 2) {
      float gu[16 * EPI_LD];     // [g(ch), u(ch), g(ch+1), u(ch+1), ...], one wait per batch
      if constexpr (EPI_LD == 4)
        tmem_ld16x4(taddr + ch * 16, taddr + 128 + ch * 16, taddr + ch * 16 + 16, taddr + 144 + ch * 16, gu);
      else
        tmem_ld16x2(taddr + ch * 16, taddr + 128 + ch * 16, gu);
#pragma unroll
      for (int b = 0; b < EPI_LD / 2; ++b) {
        const float* g = gu + 32 * b;
        const float* u = g + 16;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162 p = __floats2bfloat162_rn(silu_mul(g[2 * j], u[2 * j]), silu_mul(g[2 * j + 1], u[2 * j + 1]));
          w[(ch + b) * 8 + j] = *reinterpret_cast<uint32_t*>(&p);
        }
      }
    }
  } else {
#pragma unroll
    for (int ch = 0; ch < BN / 16; ch += EPI_LD) {
      float v[16 * EPI_LD];
      if constexpr (EPI_LD == 4)
        tmem_ld16x4(taddr + ch * 16, taddr + ch * 16 + 16, taddr + ch * 16 + 32, taddr + ch * 16 + 48, v);
      else
        tmem_ld16x2(taddr + ch * 16, taddr + ch * 16 + 16, v);
#pragma unroll
      for (int j = 0; j < 8 * EPI_LD; ++j) {
        __nv_bfloat162 p = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[ch * 8 + j] = *reinterpret_cast<uint32_t*>(&p);
      }
    }
  }
  tc_fence_before();
  release();                      // TMEM free: the MMA proceeds with the tile after next
  __nv_bfloat16* dst = valid ? orow : nullptr;
  if (MODE == MODE_GATEUP) {
    store_rows_staged<NW>(w, dst, nb * 128, 128, stage, lane);
  } else {
    if (args.fuse) flush_count(dc, pend, fwd);      // the previous tile's rows
    store_rows_staged<NW>(w, dst, nb * BN, min(BN, args.out_cols - nb * BN), stage, lane);
    if (args.fuse) {
      const int cols = min(BN, dc.d - nb * BN);
      if (valid && cols > 0) { pend.leg = leg; pend.pieces = cols; pend.nb = nb; }
    }
  }
}

// Split-K (cold experts: fewer output tiles than SMs): a unit (tile, ks) covers K blocks
// [ks·kb/split, (ks+1)·kb/split). Its fp32 partial rows go to part[(slot·split + ks)·128 + r];
// splitk_reduce_kernel then sums the partials in ks order (deterministic, independent of which
// unit finished first) and runs the final stores.
template <int MODE, int BN, typename Release>
__device__ __forceinline__ void epilogue_unit(const FfnArgs& args, const DevCtx& dc, uint32_t taddr, int split, int ks,
                                              int slot, int rloc, bool valid, __nv_bfloat16* orow, int nb,
                                              const amoe_leg& leg, uint32_t stage, int lane, uint32_t (&fwd)[2],
                                              PendCount& pend, Release release) {
  if (split <= 1) {
    epilogue_tile<MODE, BN>(args, dc, taddr, valid, orow, nb, leg, stage, lane, fwd, pend, release);
    return;
  }
  constexpr int W = (MODE == MODE_GATEUP) ? 256 : BN;      // fp32 columns per partial row
  float* mine = args.part + ((size_t)(slot * split + ks) * 128 + rloc) * W;
#pragma unroll 1
  for (int c0 = 0; c0 < W; c0 += 32) {
    float v[32];
    tmem_ld32(taddr + c0, v);
    if (valid) {
      float4* d4 = reinterpret_cast<float4*>(mine + c0);
#pragma unroll
      for (int j = 0; j < 8; ++j) d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  }
  tc_fence_before();
  release();                       // TMEM free: the MMA proceeds with the next unit
  // the fixed-order reduction and the final stores run in splitk_reduce_kernel (stream-ordered)
}

// Device-side split decision (identical in every CTA and in splitk_reduce_kernel). Split K only
// in the cold regime — every queue fits one M tile, so weight streaming dominates — and only when
// slots (CTAs or CTA pairs) would idle: fewer output tiles than slots, or up to 1.25x as many when
// the unit's fp32 partial rows are tiny (<= 16 rows per half). halves = split-K slots per tile
// (2 for a CTA pair: each CTA reduces its own 128 rows). ~3 units per slot, >= 8 K blocks per
// unit, and each unit's partial rows (rows x 1 KB) <= 1/4 of the weight bytes it streams (16 KB
// per K block per CTA): s <= 4·kb / rows. Tuned with tools/rebatch_sweep.py A/B runs
// (profiles/r01_rebatch_sweep.md): splitting with tiles >= slots, or heavy partials, was slower.
__device__ __forceinline__ int choose_split(const FfnArgs& a, int tiles, int slots, int halves, int max_m_tiles,
                                            int max_n) {
  if (!a.allow_split || tiles <= 0 || max_m_tiles > 1 || tiles * halves > kSplitSlots) return 1;
  const int rows = max(1, (max_n + halves - 1) / halves);
  if (!(tiles < slots || (4 * tiles < 5 * slots && rows <= 16))) return 1;
  int s = (3 * slots + tiles - 1) / tiles;
  s = min(s, a.k_blocks / 8);
  s = min(s, 32);
  s = min(s, kSplitUnits / (tiles * halves));
  s = min(s, 4 * a.k_blocks / rows);
  return max(s, 1);
}

// Token slots of 4 consecutive rows of queue q starting at row r0 (rows >= n use slot 0: their
// outputs are never stored).
__device__ __forceinline__ int4 gather_rows(const FfnArgs& a, const DevCtx& dc, int q, int r0, int n,
                                            const int* s_start) {
  int v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = (r0 + i < n) ? leg_of_row(a, dc, q, r0 + i, 0, s_start).token_slot : 0;
  return make_int4(v[0], v[1], v[2], v[3]);
}
template <int MODE, int BN>
__global__ void __launch_bounds__(THREADS, 1)
ffn_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA32, const FfnArgs args,
              const __grid_constant__ DevCtx dc) {
  AMOE_PDL_ENTRY();
  __shared__ unsigned long long s_fwd[2];     // legs forwarded, of which remote
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  // bars: full[STAGES], empty[STAGES], tfull[2], tempty[2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  int* s_n = reinterpret_cast<int*>(tmem_holder + 4);
  int* s_off = s_n + AMOE_MAX_GROUP;
  int* s_pre = s_off + AMOE_MAX_GROUP;   // AMOE_MAX_GROUP + 1
  int* s_start = s_pre + AMOE_MAX_GROUP + 1;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nq = args.nq;
  for (int q = tid; q < nq; q += THREADS) {
    s_n[q] = args.qinfo[q]; s_off[q] = args.qinfo[AMOE_MAX_GROUP + q]; s_start[q] = args.qinfo[2 * AMOE_MAX_GROUP + q];
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    int mm = 0;
    for (int q = 0; q < nq; ++q) {
      s_pre[q] = acc; acc += (s_n[q] + BM - 1) / BM * args.n_tiles; mm = max(mm, (s_n[q] + BM - 1) / BM);
    }
    s_pre[nq] = acc;
    s_start[AMOE_MAX_GROUP] = mm;
    int mn = 0;
    for (int q = 0; q < nq; ++q) mn = max(mn, s_n[q]);
    s_start[AMOE_MAX_GROUP + 1] = mn;
    s_fwd[0] = 0; s_fwd[1] = 0;
    for (int s = 0; s < STAGES; ++s) { mbar_init(smem_u32(&bars[s]), 1); mbar_init(smem_u32(&bars[STAGES + s]), 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(smem_u32(&bars[2 * STAGES + a]), 1); mbar_init(smem_u32(&bars[2 * STAGES + 2 + a]), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&tmA);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_holder)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  Sched sc{nq, args.n_tiles, s_pre[nq], args.group_m, s_n, s_off, s_pre};
  const int kb_n = args.k_blocks;
  const int split = choose_split(args, sc.total, gridDim.x, 1, s_start[AMOE_MAX_GROUP], s_start[AMOE_MAX_GROUP + 1]);
  const int units = sc.total * split;

  if (warp == 0 && (lane == 0 || (MODE == MODE_GATEUP && args.gather))) {
    // ===================== TMA producer (lane 0; the whole warp when A rows are gathered:
    // lane i issues the tile::gather4 of tile rows 4i..4i+3)
    int stage = 0; uint32_t phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u / split, ks = u - t * split;
      int q, m, nb;
      sc.decode(t, q, m, nb);
      const int arow = s_off[q] + m * BM;
      const CUtensorMap* wb = args.wmaps + args.wslot[q] + args.w_which;
      const int kb0 = ks * kb_n / split, kb1 = (ks + 1) * kb_n / split;
      if (MODE == MODE_GATEUP && args.gather) {
        const int4 rows4 = gather_rows(args, dc, q, m * BM + lane * 4, s_n[q], s_start);
        for (int kb = kb0; kb < kb1; ++kb) {
          const uint32_t full = smem_u32(&bars[stage]);
          const uint32_t sa = smem_u32(tiles + stage * STAGE_BYTES);
          if (lane == 0) {
            mbar_wait(smem_u32(&bars[STAGES + stage]), phase ^ 1u);
            mbar_expect_tx(full, A_BYTES + BN * BK * 2);
          }
          __syncwarp();
          tma_gather4(sa + lane * 4 * 128, &tmA, kb * BK, rows4, full);
          if (lane == 0) {
            tma_load_2d(sa + A_BYTES, wb, kb * BK, nb * 128, full);
            tma_load_2d(sa + A_BYTES + 128 * BK * 2, wb + 1, kb * BK, nb * 128, full);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
        continue;
      }
      // A partial M tile loads only its valid rows (32-row boxes); the rest of the smem tile is
      // stale and only feeds accumulator rows that are never stored. Decided per tile, in its own
      // loop: extra work between the empty-slot wait and the TMA issue delays every refill
      // (measured: ~30% of the pair kernel's throughput).
      const int rows_valid = s_n[q] - m * BM;
      const int nA = (!args.atrim || rows_valid >= BM) ? 0 : (rows_valid + 31) / 32;
      auto load_b = [&](uint32_t sb, int kb, uint32_t full) {
        if (MODE == MODE_GATEUP) {
          tma_load_2d(sb, wb, kb * BK, nb * 128, full);
          tma_load_2d(sb + 128 * BK * 2, wb + 1, kb * BK, nb * 128, full);
        } else {
          // weight maps have 128-row boxes: BN = 256 takes two loads
#pragma unroll
          for (int h = 0; h < BN / 128; ++h) tma_load_2d(sb + h * 128 * BK * 2, wb, kb * BK, nb * BN + h * 128, full);
        }
      };
      if (nA == 0) {
        for (int kb = kb0; kb < kb1; ++kb) {
          const uint32_t full = smem_u32(&bars[stage]);
          const uint32_t sa = smem_u32(tiles + stage * STAGE_BYTES);
          mbar_wait(smem_u32(&bars[STAGES + stage]), phase ^ 1u);
          mbar_expect_tx(full, A_BYTES + BN * BK * 2);
          tma_load_2d(sa, &tmA, kb * BK, arow, full);
          load_b(sa + A_BYTES, kb, full);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      } else {
        const uint32_t tx = nA * 32 * BK * 2 + BN * BK * 2;
        for (int kb = kb0; kb < kb1; ++kb) {
          const uint32_t full = smem_u32(&bars[stage]);
          const uint32_t sa = smem_u32(tiles + stage * STAGE_BYTES);
          mbar_wait(smem_u32(&bars[STAGES + stage]), phase ^ 1u);
          mbar_expect_tx(full, tx);
          for (int i = 0; i < nA; ++i) tma_load_2d(sa + i * 32 * BK * 2, &tmA32, kb * BK, arow + i * 32, full);
          load_b(sa + A_BYTES, kb, full);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ===================== MMA issuer (single thread)
    constexpr uint32_t idesc = idesc_bf16(BM, BN);
    int stage = 0; uint32_t phase = 0;
    int acc = 0; uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int ks = u % split;
      const int kb0 = ks * kb_n / split, kb1 = (ks + 1) * kb_n / split;
      mbar_wait(smem_u32(&bars[2 * STAGES + 2 + acc]), acc_phase ^ 1u);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * 256);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(smem_u32(&bars[stage]), phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(tiles + stage * STAGE_BYTES);
        const uint64_t adesc = umma_desc_sw128(sa);
        const uint64_t bdesc = umma_desc_sw128(sa + A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)   // +32 B along K inside the swizzle atom = +2 in desc units
          umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0) | (k > 0));
        umma_commit(smem_u32(&bars[STAGES + stage]));     // frees the smem stage when MMAs retire
        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
      }
      umma_commit(smem_u32(&bars[2 * STAGES + acc]));      // accumulator ready
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> registers -> global
    const int ew = warp - 4;            // TMEM lane quarter (warp % 4)
    const uint32_t stage = smem_u32(smem + STAGES * STAGE_BYTES + 4096 + ew * 4096);
    uint32_t fwd[2] = {0u, 0u};         // legs forwarded by this thread's rows, of which remote
    PendCount pend{};
    int acc = 0; uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u / split, ks = u - t * split;
      int q, m, nb;
      sc.decode(t, q, m, nb);
      epi_wait(smem_u32(&bars[2 * STAGES + acc]), acc_phase, tid, 128);
      tc_fence_after();
      const int row = m * BM + ew * 32 + lane;
      const bool valid = row < s_n[q];
      amoe_leg leg;
      __nv_bfloat16* orow = down_row_dst<MODE>(args, dc, q, row, s_off[q] + row, s_start, valid, leg);
      const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(ew * 32) << 16);
      const uint32_t tempty = smem_u32(&bars[2 * STAGES + 2 + acc]);
      epilogue_unit<MODE, BN>(args, dc, taddr, split, ks, t, ew * 32 + lane, valid, orow, nb, leg, stage, lane, fwd,
                              pend, [&] { epi_release_local(tempty, tid, 128); });
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    if (MODE == MODE_DOWN && args.fuse) {
      flush_count(dc, pend, fwd);         // the last tile's rows
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        fwd[0] += __shfl_xor_sync(0xffffffffu, fwd[0], o);
        fwd[1] += __shfl_xor_sync(0xffffffffu, fwd[1], o);
      }
      if (lane == 0) { atomicAdd(&s_fwd[0], (unsigned long long)fwd[0]); atomicAdd(&s_fwd[1], (unsigned long long)fwd[1]); }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
  if (MODE == MODE_DOWN && args.fuse && tid == 0) {
    unsigned long long* st = wsp<unsigned long long>(dc, dc.rank, dc.lay.stats);
    if (s_fwd[0]) atomicAdd(st + 2, s_fwd[0]);
    if (s_fwd[1]) atomicAdd(st + 3, s_fwd[1]);
  }
}

// ================================================================== CTA-pair variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile with UMMA M = 256.
// CTA r loads A rows [m0 + 128 r, +128) and B rows [128 r, +128) of the 256-row B operand
// (GATEUP: r = 0 -> W1 slab, r = 1 -> W3 slab; DOWN: W2 rows n0 + 128 r ...). The leader (r = 0)
// issues the MMAs, which read A and B halves from both CTAs' shared memory; each CTA's TMEM
// holds its own 128 rows x 256 fp32 columns, so the epilogue is per CTA as in the 1-CTA kernel.
// Per CTA and per K=16 step this stages 8 KB instead of 12 KB (-33 % L2->SM bytes per FLOP).
namespace tc2 {
using namespace tc;
#ifndef AMOE_STAGES2
#define AMOE_STAGES2 6
#endif
#ifndef AMOE_L2PF
#define AMOE_L2PF 0
#endif
constexpr int STAGES2 = AMOE_STAGES2;
// producer L2 prefetch distance in K blocks (0: off): the first CTA to touch an operand line
// pays the DRAM latency; a bulk-tensor L2 prefetch that many blocks ahead hides it
constexpr int L2PF = AMOE_L2PF;
constexpr int HALF_BYTES = 128 * BK * 2;                     // 16 KB
constexpr int STAGE2_BYTES = 2 * HALF_BYTES;                 // A half + B half = 32 KB
constexpr int SMEM2_BYTES = STAGES2 * STAGE2_BYTES + 4096 + EPI_STAGE_BYTES + 1024;
constexpr int BM2 = 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const void* tmap, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(dst), "l"(tmap), "r"(c0), "r"(c1), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const void* tmap, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" :: "l"(tmap), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// arrive on the barrier at this smem offset in both CTAs of the pair when the MMAs retire
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
      "}\n" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(bar_cluster) : "memory");
}

// ------------------------------------------------------------------ die-aware unit ring
// The leader's producer claims units (tile, K split) from its die's list — each die owns a
// share of every queue's N tiles, so a weight slab is streamed into one die's L2 only —
// stealing from the other die's list when its own runs out, and publishes each unit to a ring
// in both CTAs' shared memory. The leader's MMA issuer and epilogue and the peer's producer
// and epilogue consume the ring in order (4 arrivals free a slot).
constexpr int RING = 8;
__device__ __forceinline__ uint32_t smid_u32() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITC_%=;\n}\n" :: "r"(bar), "r"(parity), "r"(kSuspendNs) : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, int4 v) {
  asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};"
               :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ int4 lds_v4(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}

struct Sched2 {
  int nq, n_tiles, total, group;
  const int* n;
  const int* pre;
  __device__ __forceinline__ void decode(int t, int& q, int& m, int& nb) const {
    int lo = 0, hi = nq - 1;
    while (lo < hi) { int mid = (lo + hi + 1) >> 1; if (pre[mid] <= t) lo = mid; else hi = mid - 1; }
    q = lo;
    const int u = t - pre[q];
    const int m_tiles = (n[q] + BM2 - 1) / BM2;
    const int gsz = group * n_tiles;
    const int g = u / gsz;
    const int first_m = g * group;
    const int gm = min(m_tiles - first_m, group);
    const int r = u - g * gsz;
    m = first_m + r % gm;
    nb = r / gm;
  }
};

#ifdef AMOE_TRACE
// diagnostic build only (-DAMOE_TRACE): per-CTA timeline of the last launch of each mode,
// read with amoe_debug_ffn_trace (tools/ffn_trace.py)
__device__ unsigned long long g_ffn_trace[2][8][160];
#define FFN_TRACE(i, v) (g_ffn_trace[MODE == MODE_GATEUP ? 0 : 1][i][blockIdx.x] = (v))
#else
#define FFN_TRACE(i, v) ((void)0)
#endif

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1)
ffn_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const FfnArgs args, const __grid_constant__ DevCtx dc) {
  AMOE_PDL_ENTRY();
  if (threadIdx.x == 0) FFN_TRACE(0, globaltimer_ns());
  __shared__ unsigned long long s_fwd[2];
  __shared__ int4 s_epi_rec[1];            // die schedule: the epilogue's current unit
  __shared__ __align__(8) uint64_t s_afull[STAGES2];   // cp.async gather: A rows of a stage landed
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* tiles = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  const bool gcp = MODE == MODE_GATEUP && args.gather == 2;
  // bars: full[S], empty[S], tfull[2], tempty[2]   (full/tempty used in the leader only)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES2 + 4);
  int* s_n = reinterpret_cast<int*>(tmem_holder + 4);
  int* s_off = s_n + AMOE_MAX_GROUP;
  int* s_pre = s_off + AMOE_MAX_GROUP;
  int* s_start = s_pre + AMOE_MAX_GROUP + 1;
  // die-aware schedule: per-die tile prefix sums, the unit ring and its barriers
  int* s_pre_d = s_start + AMOE_MAX_GROUP + 4;                       // [2][AMOE_MAX_GROUP + 1]
  int4* ring = reinterpret_cast<int4*>(((reinterpret_cast<uintptr_t>(s_pre_d + 2 * (AMOE_MAX_GROUP + 1))) + 15) &
                                       ~uintptr_t(15));
  uint64_t* ring_full = reinterpret_cast<uint64_t*>(ring + RING);
  uint64_t* ring_empty = ring_full + RING;
  int* s_die = reinterpret_cast<int*>(ring_empty + RING);           // [0] = N-tile split point

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int nq = args.nq;
  for (int q = tid; q < nq; q += THREADS) {
    s_n[q] = args.qinfo[q]; s_off[q] = args.qinfo[AMOE_MAX_GROUP + q]; s_start[q] = args.qinfo[2 * AMOE_MAX_GROUP + q];
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    int mm = 0;
    for (int q = 0; q < nq; ++q) {
      s_pre[q] = acc; acc += (s_n[q] + BM2 - 1) / BM2 * args.n_tiles; mm = max(mm, (s_n[q] + BM2 - 1) / BM2);
    }
    s_pre[nq] = acc;
    s_start[AMOE_MAX_GROUP] = mm;
    int mn = 0;
    for (int q = 0; q < nq; ++q) mn = max(mn, s_n[q]);
    s_start[AMOE_MAX_GROUP + 1] = mn;
    s_fwd[0] = 0; s_fwd[1] = 0;
    // cp.async gather (gcp): a stage's full barrier also takes one arrival per CTA from its
    // relay thread (A rows landed); each CTA's s_afull collects its producer lanes' cp.async
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(smem_u32(&bars[s]), gcp ? 3 : 1);   // (one relay arrival per CTA per stage)
      mbar_init(smem_u32(&bars[STAGES2 + s]), 1);
      if (gcp) mbar_init(smem_u32(&s_afull[s]), kWarp);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&bars[2 * STAGES2 + a]), 1);
      mbar_init(smem_u32(&bars[2 * STAGES2 + 2 + a]), 2);     // one arrive per CTA of the pair
    }
    if (args.die_sched) {
      // die d owns N tiles [lo_d, hi_d) of every queue, in proportion to its SM count
      // (die_sched == 3, "dynamic": die 0's list holds every tile; both dies claim from it)
      const int tot = dc.die_cnt[0] + dc.die_cnt[1];
      const int h = args.die_sched == 3 ? args.n_tiles : (args.n_tiles * dc.die_cnt[0] + tot / 2) / tot;
      s_die[0] = h;
      for (int d = 0; d < 2; ++d) {
        const int nbd = d == 0 ? h : args.n_tiles - h;
        int a2 = 0;
        for (int q = 0; q < nq; ++q) { s_pre_d[d * (AMOE_MAX_GROUP + 1) + q] = a2; a2 += (s_n[q] + BM2 - 1) / BM2 * nbd; }
        s_pre_d[d * (AMOE_MAX_GROUP + 1) + nq] = a2;
      }
      // consumers of a published unit: leader MMA + epilogue, peer producer + epilogue (+ each
      // CTA's relay thread under the cp.async gather)
      for (int r = 0; r < RING; ++r) { mbar_init(smem_u32(&ring_full[r]), 1); mbar_init(smem_u32(&ring_empty[r]), gcp ? 6 : 4); }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&tmA);
  }
  // this CTA's weight tensor maps of every queue (a grouped launch may hold 66 of them): fetched
  // now instead of on each queue's first TMA load
  if (warp == 3)
    for (int q = lane; q < nq; q += kWarp)
      tma_prefetch(args.wmaps + args.wslot[q] + args.w_which + (MODE == MODE_GATEUP ? (int)crank : 0));
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_holder)), "r"(TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (tid == 0) FFN_TRACE(1, globaltimer_ns());
  Sched2 sc{nq, args.n_tiles, s_pre[nq], args.group_m, s_n, s_pre};
  const int kb_n = args.k_blocks;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int split = choose_split(args, sc.total, ncl, 2, s_start[AMOE_MAX_GROUP], s_start[AMOE_MAX_GROUP + 1]);
  const int units = sc.total * split;
  const bool die_sched = args.die_sched != 0;
  // unit = {q, m, nb, ks}; q < 0: no more units. Static schedule: cluster cl takes units
  // cl, cl + ncl, ... of the global raster.
  auto static_unit = [&](int it) -> int4 {
    const int u = cl + it * ncl;
    if (u >= units) return make_int4(-1, 0, 0, 0);
    const int t = u / split;
    int q, m, nb;
    sc.decode(t, q, m, nb);
    return make_int4(q, m, nb, u - t * split);
  };
  // die-local unit u of die d -> {q, m, nb, ks}: the raster of Sched2 restricted to the die's
  // N tiles [lo_d, hi_d) of every queue (measured: contiguous ranges of whole queues per die
  // kept the DRAM traffic; this split cut the Mixtral gate/up reads 5.6 -> 3.4 GB)
  auto die_units = [&](int d) -> int { return s_pre_d[d * (AMOE_MAX_GROUP + 1) + nq] * split; };
  auto die_unit = [&](int d, int u) -> int4 {
    const int* pre = s_pre_d + d * (AMOE_MAX_GROUP + 1);
    const int lo = d == 0 ? 0 : s_die[0];
    const int nbd = d == 0 ? s_die[0] : args.n_tiles - s_die[0];
    const int t = u / split;
    int qlo = 0, qhi = nq - 1;
    while (qlo < qhi) { const int mid = (qlo + qhi + 1) >> 1; if (pre[mid] <= t) qlo = mid; else qhi = mid - 1; }
    const int q = qlo;
    const int r = t - pre[q];
    const int m_tiles = (s_n[q] + BM2 - 1) / BM2;
    const int gsz = sc.group * nbd;
    const int g = r / gsz;
    const int first_m = g * sc.group;
    const int gm = min(m_tiles - first_m, sc.group);
    const int rr = r - g * gsz;
    return make_int4(q, first_m + rr % gm, lo + rr / gm, u - t * split);
  };
  // leader producer: claims are issued one unit ahead (the atomic's latency overlaps the
  // current unit's loads) and resolved — own die first, then the other die's list — into the
  // unit published to both CTAs' rings one unit ahead of its loads
  // single list (die_sched == 3): every cluster's first unit is its own index (no claim), the
  // counter hands out units ncl, ncl + 1, ... — a cluster that pre-claims its second unit at
  // the start can then never take a first unit from another (with fewer units than 2 x clusters
  // the claim-ahead alone left half the clusters idle and doubled the kernel time)
  const bool single = args.die_sched == 3;
  const int my_die = single ? 0 : (int)((dc.die_mask[smid_u32() >> 6] >> (smid_u32() & 63)) & 1ull);
  const uint32_t claim_base = single ? (uint32_t)ncl : 0u;
  int claim_d = my_die;
  uint32_t claim_u = 0;
  auto issue_claim = [&]() { claim_u = atomicAdd(args.sched + claim_d, 1u) + (claim_d == 0 ? claim_base : 0u); };
  auto resolve_claim = [&]() -> int4 {
    for (;;) {
      const int ud = die_units(claim_d);
      if (claim_u < (uint32_t)ud) return die_unit(claim_d, (int)claim_u);
      if (single || claim_d != my_die) return make_int4(-1, 0, 0, 0);   // no list left
      claim_d = 1 - my_die;                                     // steal
      issue_claim();
    }
  };
  auto publish = [&](int it, int4 rec) {
    const int slot = it % RING;
    mbar_wait_cluster(smem_u32(&ring_empty[slot]), ((it / RING) & 1) ^ 1u);
    // the peer's copy: an asynchronous remote store that completes the peer's barrier phase
    // itself (st.async + expect_tx): no cluster-scope release fence on the producer's path
    const uint32_t pf = mapa(smem_u32(&ring_full[slot]), 1);
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], 16;" :: "r"(pf) : "memory");
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.s32 [%0], {%1, %2, %3, %4}, [%5];"
                 :: "r"(mapa(smem_u32(&ring[slot]), 1)), "r"(rec.x), "r"(rec.y), "r"(rec.z), "r"(rec.w), "r"(pf)
                 : "memory");
    ring[slot] = rec;                                              // the leader's copy: CTA scope
    mbar_arrive(smem_u32(&ring_full[slot]));
  };
  int4 next_unit = make_int4(-1, 0, 0, 0);
  auto claim_publish = [&](int it) -> int4 {
    if (it == 0) {                         // unit 0 now; the claim for unit 1 in flight
      if (single) {
        claim_u = (uint32_t)cl;
      } else {
        issue_claim();
      }
      next_unit = resolve_claim();
      publish(0, next_unit);
      if (next_unit.x >= 0) {
        if (single && units <= ncl) claim_u = ~0u;   // one round: no second unit to claim
        else issue_claim();
      }
    }
    return next_unit;                      // published one unit ago
  };
  // ... and, once the current unit's first stage is issued (the bookkeeping stays off the
  // load pipeline's critical path), resolve and publish unit it + 1 and issue the next claim
  auto advance = [&](int it) {
    next_unit = resolve_claim();
    publish(it + 1, next_unit);
    if (next_unit.x >= 0) issue_claim();
  };
  // (claim_u = ~0u resolves to the end record without an atomic)
  // every other role (one thread): take unit `it` from this CTA's ring, free the slot. The free
  // is a relaxed arrive ordered after the record load by a dependency on its value: a release
  // arrive would first drain this thread's outstanding global stores (the epilogue's output
  // rows), stalling the epilogue for microseconds per unit.
  auto ring_get = [&](int it) -> int4 {
    const int slot = it % RING;
    // CTA-scope waits: the leader's copy comes from a same-CTA producer, the peer's through the
    // barrier's own transaction count (st.async), as TMA data does
    mbar_wait(smem_u32(&ring_full[slot]), (it / RING) & 1);
    const int4 rec = lds_v4(smem_u32(&ring[slot]));
    // (rec.x is a queue index or -1, never INT_MIN: the select is 0, but the address depends on
    // the loaded value, so the arrive cannot be performed before the load)
    const uint32_t eb = mapa(smem_u32(&ring_empty[slot]), 0) + (rec.x == INT_MIN ? 8u : 0u);
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(eb) : "memory");
    return rec;
  };

  if (gcp && warp == 0) {
    // ===================== producer with the re-batch gather fused (both CTAs, whole warp):
    // this CTA's 128 A rows of a stage are the legs' x rows, copied by cp.async 16-B chunks
    // straight from x[token_slot] into the 128-B-swizzled stage (lanes 8j..8j+7 write the 8
    // chunks of one row: conflict-free), rows >= n zero-filled; the lanes' copies arrive on
    // s_afull when they land (noinc), and the relay thread hands the stage to the leader. The B
    // half is a TMA load onto the leader's full barrier, as in the tiled producer. The token
    // slots of the next unit's rows are loaded while the current unit streams (no drain-to-GEMM
    // bubble per unit). Every A row is re-read by each N tile of its raster group, from L2: the
    // same L2 traffic as the materialised tile, without the gather kernel's HBM round trip
    // (2·d·2 bytes per leg) — single GPU only (peer rows would cross NVLink once per N tile).
    const char* xb = reinterpret_cast<const char*>(dc.peer[dc.rank] + dc.lay.x);
    const uint32_t rowbytes = (uint32_t)dc.d * 2u;
    const int rsub = lane >> 3, csub = lane & 7;
    const amoe_leg* rings = reinterpret_cast<const amoe_leg*>(dc.peer[dc.rank] + dc.lay.rings);
    auto bcast = [&](int4 u) -> int4 {
      u.x = __shfl_sync(0xffffffffu, u.x, 0); u.y = __shfl_sync(0xffffffffu, u.y, 0);
      u.z = __shfl_sync(0xffffffffu, u.z, 0); u.w = __shfl_sync(0xffffffffu, u.w, 0);
      return u;
    };
    // token slot of rows lane + 32 j of this CTA's half of unit u's M tile (-1: row >= n)
    auto slots_of = [&](int4 u, int (&sl)[4]) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = u.y * BM2 + (int)crank * 128 + lane + 32 * j;
        sl[j] = -1;
        if (u.x >= 0 && row < s_n[u.x])
          sl[j] = rings[(uint64_t)(args.wslot[u.x] / 3) * dc.ring_cap +
                        (((uint32_t)s_start[u.x] + (uint32_t)row) & dc.ring_mask)].token_slot;
      }
    };
    int4 U = make_int4(-1, 0, 0, 0);
    if (lane == 0) U = !die_sched ? static_unit(0) : leader ? claim_publish(0) : ring_get(0);
    U = bcast(U);
    int sl[4];
    slots_of(U, sl);
    int stage = 0; uint32_t phase = 0;
    for (int it = 0; U.x >= 0; ++it) {
      const int q = U.x, nb = U.z, ks = U.w;
      const int kb0 = ks * kb_n / split, kb1 = (ks + 1) * kb_n / split;
      const CUtensorMap* bmap = args.wmaps + args.wslot[q] + args.w_which + crank;
      const int brow = nb * 128;
      int4 Un = make_int4(-1, 0, 0, 0);
      int sn[4] = {-1, -1, -1, -1};
      for (int kb = kb0; kb < kb1; ++kb) {
        const uint32_t full_leader = mapa(smem_u32(&bars[stage]), 0);
        const uint32_t sa = smem_u32(tiles + stage * STAGE2_BYTES);
        if (lane == 0) {
          mbar_wait(smem_u32(&bars[STAGES2 + stage]), phase ^ 1u);
          if (leader) mbar_expect_tx(smem_u32(&bars[stage]), 2 * HALF_BYTES);   // the two B halves
          tma_load_2d_pair(sa + HALF_BYTES, bmap, kb * BK, brow, full_leader);
        }
        __syncwarp();
        // this lane's 32 chunks: 16-B chunk csub of rows 4u + rsub (whole 128-B lines per
        // instruction); row r's slot lives in lane r % 32, register r / 32
        const char* src = xb + (uint64_t)kb * (BK * 2) + csub * 16;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int row = 4 * u + rsub;
          const int sv = __shfl_sync(0xffffffffu, sl[u >> 3], row & 31);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                       :: "r"(sa + (uint32_t)row * 128u + ((uint32_t)(csub ^ (row & 7)) << 4)),
                          "l"(src + (sv < 0 ? 0u : (uint32_t)sv * rowbytes)), "r"(sv < 0 ? 0u : 16u) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(smem_u32(&s_afull[stage])) : "memory");
        if (kb == kb0) {
          // the next unit (the leader resolves and publishes it here, as the tiled producer
          // does) and its rows' token slots, in flight while this unit streams
          if (lane == 0) {
            if (!die_sched) Un = static_unit(it + 1);
            else if (leader) { advance(it); Un = next_unit; }
            else Un = ring_get(it + 1);
          }
          Un = bcast(Un);
          slots_of(Un, sn);
        }
        if (++stage == STAGES2) { stage = 0; phase ^= 1u; }
      }
      U = Un;
#pragma unroll
      for (int j = 0; j < 4; ++j) sl[j] = sn[j];
    }
  } else if (gcp && warp == 3 && lane == 0) {
    // ===================== relay (both CTAs): a stage's A rows landed (every producer lane's
    // cp.async arrived on s_afull) -> order them for the tensor core (generic -> async proxy)
    // and arrive on the leader's full barrier. Walks the same units as the producer.
    // The arrive is RELAXED: a release at cluster scope compiles to MEMBAR.ALL.GPU, which cost
    // ~1.5 us per stage here (ncu: the relay's membar stalls held the gate/up GEMM at 46 % of
    // the tensor pipe). The copies are complete (observed through s_afull) and the proxy fence
    // has made them visible to the async proxy before the arrive is issued.
    int stage = 0; uint32_t phase = 0;
    const uint32_t full0 = mapa(smem_u32(&bars[0]), 0);
    for (int it = 0;; ++it) {
      const int4 U = die_sched ? ring_get(it) : static_unit(it);
      if (U.x < 0) break;
      const int kb0 = U.w * kb_n / split, kb1 = (U.w + 1) * kb_n / split;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(smem_u32(&s_afull[stage]), phase);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];"
                     :: "r"(full0 + (uint32_t)stage * 8u) : "memory");
        if (++stage == STAGES2) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 0 && (lane == 0 || (MODE == MODE_GATEUP && args.gather))) {
    // ===================== TMA producer (both CTAs): own A half + own B half, bytes land on
    // the leader's full barrier (whole warp when A rows are gathered: lane i -> rows 4i..4i+3)
    int stage = 0; uint32_t phase = 0;
    const bool gw = MODE == MODE_GATEUP && args.gather;     // whole warp in this branch
    for (int it = 0;; ++it) {
      int4 U = make_int4(-1, 0, 0, 0);
      if (lane == 0) U = !die_sched ? static_unit(it) : leader ? claim_publish(it) : ring_get(it);
      if (gw) {
        U.x = __shfl_sync(0xffffffffu, U.x, 0); U.y = __shfl_sync(0xffffffffu, U.y, 0);
        U.z = __shfl_sync(0xffffffffu, U.z, 0); U.w = __shfl_sync(0xffffffffu, U.w, 0);
      }
      if (U.x < 0) break;
      const int q = U.x, m = U.y, nb = U.z, ks = U.w;
      const int kb0 = ks * kb_n / split, kb1 = (ks + 1) * kb_n / split;
      const int arow = s_off[q] + m * BM2 + (int)crank * 128;
      const CUtensorMap* wb = args.wmaps + args.wslot[q] + args.w_which;
      const CUtensorMap* bmap = (MODE == MODE_GATEUP) ? wb + crank : wb;
      const int brow = (MODE == MODE_GATEUP) ? nb * 128 : nb * 256 + (int)crank * 128;
      if (MODE == MODE_GATEUP && args.gather) {
        const int4 rows4 = gather_rows(args, dc, q, m * BM2 + (int)crank * 128 + lane * 4, s_n[q], s_start);
        for (int kb = kb0; kb < kb1; ++kb) {
          const uint32_t full_leader = mapa(smem_u32(&bars[stage]), 0);
          const uint32_t sa = smem_u32(tiles + stage * STAGE2_BYTES);
          if (lane == 0) {
            mbar_wait(smem_u32(&bars[STAGES2 + stage]), phase ^ 1u);
            if (leader) mbar_expect_tx(smem_u32(&bars[stage]), 2 * STAGE2_BYTES);
          }
          __syncwarp();
          tma_gather4_pair(sa + lane * 4 * 128, &tmA, kb * BK, rows4, full_leader);
          if (lane == 0) tma_load_2d_pair(sa + HALF_BYTES, bmap, kb * BK, brow, full_leader);
          if (++stage == STAGES2) { stage = 0; phase ^= 1u; }
        }
        if (lane == 0 && die_sched && leader) advance(it);
        continue;
      }
      // Full tiles only: trimming partial M tiles to their valid rows (as the 1-CTA producer
      // does) measured ~15-25% slower here even when no tile was partial, and an out-of-line
      // trimmed loop for the cold (split-K) units gained nothing measurable
      // (profiles/r01_pair_regression.md).
      for (int kb = kb0; kb < kb1; ++kb) {
        const uint32_t full_leader = mapa(smem_u32(&bars[stage]), 0);
        const uint32_t sa = smem_u32(tiles + stage * STAGE2_BYTES);
        mbar_wait(smem_u32(&bars[STAGES2 + stage]), phase ^ 1u);
        if (leader) mbar_expect_tx(smem_u32(&bars[stage]), 2 * STAGE2_BYTES);
        tma_load_2d_pair(sa, &tmA, kb * BK, arow, full_leader);
        tma_load_2d_pair(sa + HALF_BYTES, bmap, kb * BK, brow, full_leader);
        if (L2PF > 0 && kb + L2PF < kb1) {
          tma_prefetch_l2(&tmA, (kb + L2PF) * BK, arow);
          tma_prefetch_l2(bmap, (kb + L2PF) * BK, brow);
        }
        if (++stage == STAGES2) { stage = 0; phase ^= 1u; }
        if (kb == kb0 && die_sched && leader) advance(it);
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ===================== MMA issuer (leader CTA, single thread), UMMA 256 x 256 x 16
    constexpr uint32_t idesc = idesc_bf16(BM2, 256);
    int stage = 0; uint32_t phase = 0;
    int acc = 0; uint32_t acc_phase = 0;
#ifdef AMOE_TRACE
    unsigned long long t_wait_full = 0, t_wait_tmem = 0, t_ring = 0;
#endif
    for (int it = 0;; ++it) {
#ifdef AMOE_TRACE
      const unsigned long long tr0 = globaltimer_ns();
#endif
      const int4 U = die_sched ? ring_get(it) : static_unit(it);
#ifdef AMOE_TRACE
      t_ring += globaltimer_ns() - tr0;
      if (U.x < 0) { FFN_TRACE(3, globaltimer_ns()); FFN_TRACE(4, it); FFN_TRACE(5, t_wait_full); FFN_TRACE(6, t_wait_tmem); FFN_TRACE(7, t_ring); }
#endif
      if (U.x < 0) break;
      const int ks = U.w;
      const int kb0 = ks * kb_n / split, kb1 = (ks + 1) * kb_n / split;
#ifdef AMOE_TRACE
      const unsigned long long tt0 = globaltimer_ns();
#endif
      mbar_wait(smem_u32(&bars[2 * STAGES2 + 2 + acc]), acc_phase ^ 1u);
#ifdef AMOE_TRACE
      t_wait_tmem += globaltimer_ns() - tt0;
#endif
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * 256);
      for (int kb = kb0; kb < kb1; ++kb) {
#ifdef AMOE_TRACE
        const unsigned long long tf0 = globaltimer_ns();
#endif
        if (gcp) {
          // A rows written by both CTAs' cp.async (generic proxy, fenced by the relays)
          mbar_wait_cluster(smem_u32(&bars[stage]), phase);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        } else {
          mbar_wait(smem_u32(&bars[stage]), phase);
        }
#ifdef AMOE_TRACE
        const unsigned long long tf1 = globaltimer_ns();
        t_wait_full += tf1 - tf0;
        if (it == 0 && kb == kb0) FFN_TRACE(2, tf1);
#endif
        tc_fence_after();
        const uint32_t sa = smem_u32(tiles + stage * STAGE2_BYTES);
        const uint64_t adesc = umma_desc_sw128(sa);
        const uint64_t bdesc = umma_desc_sw128(sa + HALF_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma_bf16_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb > kb0) | (k > 0));
        umma_commit_pair(smem_u32(&bars[STAGES2 + stage]));       // frees the stage in both CTAs
        if (++stage == STAGES2) { stage = 0; phase ^= 1u; }
      }
      umma_commit_pair(smem_u32(&bars[2 * STAGES2 + acc]));        // accumulators ready in both
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs): own 128 rows
    const int ew = warp - 4;
    const uint32_t stage = smem_u32(smem + STAGES2 * STAGE2_BYTES + 4096 + ew * 4096);
    uint32_t fwd[2] = {0u, 0u};
    PendCount pend{};
    int acc = 0; uint32_t acc_phase = 0;
    const uint32_t tempty_leader0 = mapa(smem_u32(&bars[2 * STAGES2 + 2]), 0);
    for (int it = 0;; ++it) {
      int4 U;
      if (die_sched) {
        if (tid == 128) s_epi_rec[0] = ring_get(it);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        U = s_epi_rec[0];
      } else {
        U = static_unit(it);
      }
      if (U.x < 0) break;
      const int q = U.x, m = U.y, nb = U.z, ks = U.w;
      const int t = s_pre[q] + nb;           // split units: the tile's global index (m = 0)
      epi_wait(smem_u32(&bars[2 * STAGES2 + acc]), acc_phase, tid, 128);
      tc_fence_after();
      const int row = m * BM2 + (int)crank * 128 + ew * 32 + lane;
      const bool valid = row < s_n[q];
      amoe_leg leg;
      __nv_bfloat16* orow = down_row_dst<MODE>(args, dc, q, row, s_off[q] + row, s_start, valid, leg);
      const uint32_t taddr = tmem_base + (uint32_t)(acc * 256) + ((uint32_t)(ew * 32) << 16);
      const uint32_t tempty = tempty_leader0 + (uint32_t)(acc * 8);
      // each CTA's half tile is its own split-K slot: 2 t + crank
      epilogue_unit<MODE, 256>(args, dc, taddr, split, ks, 2 * t + (int)crank, ew * 32 + lane, valid, orow, nb, leg,
                               stage, lane, fwd, pend, [&] {
                                 __syncwarp();
                                 asm volatile("bar.sync 1, 128;" ::: "memory");
                                 if (tid == 128) mbar_arrive_cluster(tempty);
                               });
      if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
    }
    if (MODE == MODE_DOWN && args.fuse) {
      flush_count(dc, pend, fwd);         // the last tile's rows
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        fwd[0] += __shfl_xor_sync(0xffffffffu, fwd[0], o);
        fwd[1] += __shfl_xor_sync(0xffffffffu, fwd[1], o);
      }
      if (lane == 0) { atomicAdd(&s_fwd[0], (unsigned long long)fwd[0]); atomicAdd(&s_fwd[1], (unsigned long long)fwd[1]); }
    }
  }
  if (die_sched && leader && tid == 0) {
    // every cluster has claimed its last unit before it gets here; the last one resets the
    // claim counters for the next launch (stream-ordered)
    if (atomicAdd(args.sched + 2, 1u) == (uint32_t)(ncl - 1)) {
      args.sched[0] = 0; args.sched[1] = 0; args.sched[2] = 0;
      __threadfence();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
#ifdef AMOE_TRACE
  if (tid == 0 && !leader) FFN_TRACE(3, globaltimer_ns());   // follower CTA: end time in slot 3
#endif
  if (MODE == MODE_DOWN && args.fuse && tid == 0) {
    unsigned long long* st = wsp<unsigned long long>(dc, dc.rank, dc.lay.stats);
    if (s_fwd[0]) atomicAdd(st + 2, s_fwd[0]);
    if (s_fwd[1]) atomicAdd(st + 3, s_fwd[1]);
  }
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}
}  // namespace tc2

// ================================================================== split-K reduction
// Recomputes the GEMM's (device-side) split decision from the same inputs; a no-op when the GEMM
// did not split. One warp per valid output row of a split tile: partials summed in ks order
// (coalesced fp32 loads), then the same final stores as the unsplit epilogue: SwiGLU -> act, or
// bf16 -> out / home pool + leg-piece count (fused forward).
template <int MODE, int BN, bool PAIR>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const FfnArgs args, const __grid_constant__ DevCtx dc,
                                                            int slots) {
  AMOE_PDL_ENTRY();
  constexpr int BMx = PAIR ? 256 : 128;
  constexpr int HALVES = PAIR ? 2 : 1;
  constexpr int W = (MODE == MODE_GATEUP) ? 256 : BN;        // partial row width (fp32)
  constexpr int CPL = (MODE == MODE_GATEUP ? 128 : BN) / 32;  // output columns per lane
  __shared__ int s_n[AMOE_MAX_GROUP], s_off[AMOE_MAX_GROUP], s_start[AMOE_MAX_GROUP], s_pre[AMOE_MAX_GROUP + 1];
  __shared__ int s_mmax, s_nmax;
  __shared__ int s_rpre[AMOE_MAX_GROUP + 1];   // prefix of valid (tile, row) items per queue
  const int nq = args.nq;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    s_n[q] = args.qinfo[q]; s_off[q] = args.qinfo[AMOE_MAX_GROUP + q]; s_start[q] = args.qinfo[2 * AMOE_MAX_GROUP + q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    int mm = 0;
    for (int q = 0; q < nq; ++q) {
      s_pre[q] = acc; acc += (s_n[q] + BMx - 1) / BMx * args.n_tiles; mm = max(mm, (s_n[q] + BMx - 1) / BMx);
    }
    s_pre[nq] = acc;
    s_mmax = mm;
    int mn = 0;
    for (int q = 0; q < nq; ++q) mn = max(mn, s_n[q]);
    s_nmax = mn;
    int ri = 0;
    for (int q = 0; q < nq; ++q) { s_rpre[q] = ri; ri += s_n[q] * args.n_tiles; }
    s_rpre[nq] = ri;
  }
  __syncthreads();
  const int total = s_pre[nq];
  const int split = choose_split(args, total, slots, HALVES, s_mmax, s_nmax);
  if (split <= 1) return;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  // a split launch has every queue in one M tile (m = 0), so tile t = pre[q] + nb: only the
  // valid rows (q, nb, row < n_q) are visited
  const int items = s_rpre[nq];
  for (int it = gw; it < items; it += nw) {
    int lo = 0, hi = nq - 1;
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (s_rpre[mid] <= it) lo = mid; else hi = mid - 1; }
    const int q = lo;
    const int r0 = it - s_rpre[q];
    const int nb = r0 / s_n[q], row = r0 - nb * s_n[q];
    const int t = s_pre[q] + nb;
    const int h = row / 128, r = row - h * 128;
    const int slot = PAIR ? 2 * t + h : t;
    const float* base = args.part + ((size_t)slot * split * 128 + r) * W;
    const int grow = s_off[q] + row;
    if (MODE == MODE_GATEUP) {
      const int c = lane * CPL;
      float g[CPL], u[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) { g[j] = 0.f; u[j] = 0.f; }
      // partials summed in ks order; loads issued 4 splits at a time (latency, not bandwidth)
      for (int s0 = 0; s0 < split; s0 += 4) {
        float4 a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (s0 + i < split) {
            const float* p = base + (size_t)(s0 + i) * 128 * W;
            a[i] = *reinterpret_cast<const float4*>(p + c);
            b[i] = *reinterpret_cast<const float4*>(p + 128 + c);
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (s0 + i < split) {
            g[0] += a[i].x; g[1] += a[i].y; g[2] += a[i].z; g[3] += a[i].w;
            u[0] += b[i].x; u[1] += b[i].y; u[2] += b[i].z; u[3] += b[i].w;
          }
      }
      __nv_bfloat162 o[2];
      o[0] = __floats2bfloat162_rn(silu_mul(g[0], u[0]), silu_mul(g[1], u[1]));
      o[1] = __floats2bfloat162_rn(silu_mul(g[2], u[2]), silu_mul(g[3], u[3]));
      *reinterpret_cast<uint2*>(args.out + (uint64_t)grow * args.out_ld + nb * 128 + c) = *reinterpret_cast<uint2*>(o);
    } else {
      const int c = lane * CPL;
      float v[CPL];
#pragma unroll
      for (int j = 0; j < CPL; ++j) v[j] = 0.f;
      for (int s0 = 0; s0 < split; s0 += 4) {
        float4 a[4][CPL / 4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (s0 + i < split) {
            const float* p = base + (size_t)(s0 + i) * 128 * W + c;
#pragma unroll
            for (int j = 0; j < CPL / 4; ++j) a[i][j] = *reinterpret_cast<const float4*>(p + 4 * j);
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (s0 + i < split) {
#pragma unroll
            for (int j = 0; j < CPL / 4; ++j) {
              v[4 * j] += a[i][j].x; v[4 * j + 1] += a[i][j].y; v[4 * j + 2] += a[i][j].z; v[4 * j + 3] += a[i][j].w;
            }
          }
      }
      amoe_leg leg;
      __nv_bfloat16* orow = down_row_dst<MODE>(args, dc, q, row, grow, s_start, true, leg);
      const int col = nb * BN + c;
      if (col < args.out_cols) {
#pragma unroll
        for (int j = 0; j < CPL; j += 4) {
          __nv_bfloat162 o[2];
          o[0] = __floats2bfloat162_rn(v[j], v[j + 1]);
          o[1] = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
          *reinterpret_cast<uint2*>(orow + col + j) = *reinterpret_cast<uint2*>(o);
        }
      }
      if (args.fuse) {
        fence_sc(dc.G > 1);            // every lane's row stores before the piece count
        __syncwarp();
        if (lane == 0) {
          const int cols = min(BN, dc.d - nb * BN);
          if (cols > 0) leg_pieces_done(dc, leg.home, leg.token_slot, leg.k, (uint32_t)cols);
          if (nb == 0) {
            unsigned long long* st = wsp<unsigned long long>(dc, dc.rank, dc.lay.stats);
            atomicAdd(st + 2, 1ull);
            if (leg.home != dc.rank) atomicAdd(st + 3, 1ull);
          }
        }
      }
    }
  }
}

}  // namespace tc

// ------------------------------------------------------------------ launchers


// ================================================================== SM -> die map
// B200 is two dies; each die's L2 caches its own half of the address space (2 KB interleave),
// and an SM reaches the other die's L2 over the die-to-die fabric (measured here: 28-cycle
// longer hits; tools/die_probe.cu). One CTA per SM times dependent L2 hits to NL lines; SMs of
// one die agree on which lines are near. The map is yield-dependent, so it is measured at run
// time (once per device) and used to give each die's CTA pairs their own share of the weight
// slabs (die-aware FFN schedule).
namespace probe {
constexpr int NL = 128;
constexpr int REP = 16;
__global__ void die_probe_kernel(const uint32_t* buf, uint32_t* lat, int* smids) {
  if (threadIdx.x != 0) return;
  int sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  smids[blockIdx.x] = sm;
  const uint32_t zero = buf[NL * 512 + 7];
  uint32_t v = 0;
  for (int i = 0; i < NL; ++i) {          // warm: every line into L2
    uint32_t w;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(w) : "l"(buf + i * 512) : "memory");
    v |= w;
  }
  for (int i = 0; i < NL; ++i) {
    const uint32_t* base = buf + i * 512;
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
    for (int r = 0; r < REP; ++r)
      asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(base + (v & zero)) : "memory");
    asm volatile("{\n.reg .u64 t;\nmov.u64 t, %%clock64;\nadd.u64 %0, t, %1;\n}"
                 : "=l"(t1) : "l"((uint64_t)(v & zero)) : "memory");
    lat[blockIdx.x * NL + i] = (uint32_t)((t1 - t0) / REP);
  }
}
}  // namespace probe

int die_map(uint64_t mask[4], int counts[2]);
}  // namespace amoe

#ifdef AMOE_TRACE
// [mode][slot][cta]: 0 entry, 1 setup done, 2 first stage full (leader), 3 MMA done (leader) /
// pair end (follower), 4 units (leader), 5/6/7 MMA issuer's ns waiting on full stages / TMEM /
// the unit ring (leader)
extern "C" amoe_status amoe_debug_ffn_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, amoe::tc::tc2::g_ffn_trace, sizeof(amoe::tc::tc2::g_ffn_trace)) == cudaSuccess ? AMOE_OK
                                                                                                    : AMOE_ECUDA;
}
#endif

extern "C" amoe_status amoe_die_info(int32_t counts[2]) {
  if (!counts) return AMOE_EINVAL;
  uint64_t mask[4];
  int c[2];
  amoe::die_map(mask, c);
  counts[0] = c[0];
  counts[1] = c[1];
  return AMOE_OK;
}

namespace amoe {
int die_map(uint64_t mask[4], int counts[2]) {
  static int cached_dev = -1;
  static uint64_t c_mask[4];
  static int c_cnt[2];
  int dev = 0;
  cudaGetDevice(&dev);
  if (cached_dev != dev) {
    c_mask[0] = c_mask[1] = c_mask[2] = c_mask[3] = 0;
    c_cnt[0] = c_cnt[1] = 0;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    c_cnt[0] = nsm;
    const char* env = getenv("AMOE_DIE_PROBE");
    uint32_t *buf = nullptr, *lat = nullptr;
    int* sms = nullptr;
    bool ok = (!env || env[0] != '0') && nsm <= 256 &&
              cudaMalloc(&buf, probe::NL * 2048 + 4096) == cudaSuccess &&
              cudaMalloc(&lat, (size_t)nsm * probe::NL * 4) == cudaSuccess &&
              cudaMalloc(&sms, (size_t)nsm * 4) == cudaSuccess &&
              cudaMemset(buf, 0, probe::NL * 2048 + 4096) == cudaSuccess &&
              cudaFuncSetAttribute(probe::die_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   200 * 1024) == cudaSuccess;
    std::vector<uint32_t> L((size_t)nsm * probe::NL);
    std::vector<int> S(nsm);
    if (ok) {
      probe::die_probe_kernel<<<nsm, 32, 200 * 1024>>>(buf, lat, sms);    // one CTA per SM
      ok = cudaDeviceSynchronize() == cudaSuccess &&
           cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
           cudaMemcpy(S.data(), sms, S.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    if (buf) cudaFree(buf);
    if (lat) cudaFree(lat);
    if (sms) cudaFree(sms);
    cudaGetLastError();
    if (ok) {
      // per SM: which lines are near (below the midpoint of its own min / max); SMs are then
      // split by agreement with SM 0's pattern, refined once against each group's majority
      const int NLn = probe::NL;
      std::vector<std::vector<char>> near(nsm, std::vector<char>(NLn));
      for (int b = 0; b < nsm; ++b) {
        uint32_t lo = ~0u, hi = 0;
        for (int i = 0; i < NLn; ++i) { lo = std::min(lo, L[b * NLn + i]); hi = std::max(hi, L[b * NLn + i]); }
        for (int i = 0; i < NLn; ++i) near[b][i] = 2 * L[b * NLn + i] < lo + hi;
      }
      std::vector<int> grp(nsm);
      for (int b = 0; b < nsm; ++b) {
        int agree = 0;
        for (int i = 0; i < NLn; ++i) agree += near[b][i] == near[0][i];
        grp[b] = agree >= NLn / 2 ? 0 : 1;
      }
      std::vector<char> cons(NLn);                      // group 0's majority pattern
      for (int i = 0; i < NLn; ++i) {
        int v = 0, n = 0;
        for (int b = 0; b < nsm; ++b)
          if (grp[b] == 0) { v += near[b][i]; ++n; }
        cons[i] = 2 * v >= n;
      }
      int cnt[2] = {0, 0};
      uint64_t m[4] = {0, 0, 0, 0};
      bool clean = true;
      std::vector<char> seen(256, 0);
      for (int b = 0; b < nsm; ++b) {
        int agree = 0;
        for (int i = 0; i < NLn; ++i) agree += near[b][i] == cons[i];
        if (10 * agree > 3 * NLn && 10 * agree < 7 * NLn) clean = false;   // ambiguous SM
        const int die = 2 * agree >= NLn ? 0 : 1;
        const int smid = S[b];
        if (smid < 0 || smid >= 256 || seen[smid]) { clean = false; continue; }
        seen[smid] = 1;
        cnt[die] += 1;
        if (die) m[smid >> 6] |= 1ull << (smid & 63);
      }
      if (clean && cnt[0] >= nsm / 4 && cnt[1] >= nsm / 4) {
        for (int i = 0; i < 4; ++i) c_mask[i] = m[i];
        c_cnt[0] = cnt[0];
        c_cnt[1] = cnt[1];
      }
    }
    cached_dev = dev;
  }
  for (int i = 0; i < 4; ++i) mask[i] = c_mask[i];
  counts[0] = c_cnt[0];
  counts[1] = c_cnt[1];
  return c_cnt[1] > 0;
}

// part 1: gate/up + SwiGLU -> act; part 2: down -> out, or (fuse) straight into the home pools.
// gathered: A rows of part 1 come from x by token slot (tm_tile is then the x map, box {64, 1})
// and both parts read the drained legs from the rings (no gather kernel, no meta copy).
// tm_*32: the same tensors with 32-row boxes (partial M tiles load only their valid rows).
int launch_ffn_tc(const DevCtx& c, const FfnLaunch& f, const CUtensorMap& tm_tile, const CUtensorMap& tm_act,
                  const CUtensorMap& tm_tile32, const CUtensorMap& tm_act32,
                  void* act, void* out, const amoe_leg* meta, int fuse, int gathered, int num_sms, cudaStream_t s,
                  int part) {
  using namespace tc;
#ifdef AMOE_TRACE
  if (const char* g = getenv("AMOE_TRACE_GRID")) num_sms = std::min(num_sms, atoi(g));   // diagnostic
#endif
  // the smem attribute is per device: contexts on several devices of one process (peer
  // workspaces, amoe_import_peers) each need it set on their own device
  static bool attr_done[64] = {false};
  int dev_id = 0;
  cudaGetDevice(&dev_id);
  if (dev_id < 0 || dev_id >= 64) dev_id = 0;
  if (!attr_done[dev_id]) {
    cudaFuncSetAttribute(ffn_tc_kernel<MODE_GATEUP, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(ffn_tc_kernel<MODE_DOWN, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(ffn_tc_kernel<MODE_DOWN, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(tc2::ffn_tc2_kernel<MODE_GATEUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM2_BYTES);
    cudaFuncSetAttribute(tc2::ffn_tc2_kernel<MODE_DOWN>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM2_BYTES);
    attr_done[dev_id] = true;
  }
  FfnArgs a{};
  a.nq = f.nq;
  a.qinfo = f.qinfo;
  a.wmaps = f.wmaps;
  a.meta = meta;
  a.part = reinterpret_cast<float*>(c.peer[c.rank] + c.lay.split_part);
  a.cnt = reinterpret_cast<uint32_t*>(c.peer[c.rank] + c.lay.split_cnt);
  const char* es = getenv("AMOE_SPLITK");
  a.allow_split = es ? (es[0] == '1') : 1;
  a.sched = reinterpret_cast<uint32_t*>(c.peer[c.rank] + c.lay.sched);
    const char* et = getenv("AMOE_ATRIM");
  a.atrim = et ? (et[0] == '1') : 1;
  a.ring_legs = gathered ? 1 : 0;
  a.gather = (part == 1) ? gathered : 0;
  for (int q = 0; q < f.nq; ++q) a.wslot[q] = f.wslot[q];
  // CTA-pair kernels need d % 256 == 0 and an even grid; AMOE_FFN_1CTA=1 forces 1-CTA, =0 pairs
  const char* ev = getenv("AMOE_FFN_1CTA");
  const bool force1 = ev ? ev[0] == '1' : kDefault1Cta;
  // cold launches (every queue <= 128 rows, by the caller's hint) run the 1-CTA kernels: their
  // 4 stages hold 128 KB of weights in flight per SM (the pair's 6 stages hold 96 KB next to the
  // token rows), and grouped cold experts stream at 0.82-0.93 of the HBM roofline instead of
  // 0.70-0.77 (profiles/r01_rebatch_sweep.md)
  const bool cold = f.rows_hint > 0 && f.rows_hint <= 128 && !gathered;
  const bool pair = !force1 && !cold && c.d % 256 == 0 && num_sms >= 2;
  // choose_split never splits a launch whose largest queue spans two M tiles: with the exact
  // drain counts known (amoe_run's pipelined picks) the no-op reduction launch is skipped
  const bool reduce = f.exact_max_n < 0 || f.exact_max_n <= (pair ? 256 : 128);
  const int bn = pair ? 256 : ((c.d % 256 == 0) ? 256 : 128);
  if (!pair && a.gather == 2) a.gather = 1;   // the cp.async gather is built into the pair kernel only
  if (part == 1) {            // N tiles of 128 ff-columns (x2: gate and up)
    a.n_tiles = c.ff / 128;
    a.k_blocks = c.d / BK;
    a.out_ld = c.ff;
    a.out_cols = c.ff;
    a.w_which = 0;
    a.out = reinterpret_cast<__nv_bfloat16*>(act);
  } else {                    // N tiles of bn model columns
    a.n_tiles = c.d / bn;
    a.k_blocks = c.ff / BK;
    a.out_ld = c.d;
    a.out_cols = c.d;
    a.w_which = 2;
    a.out = reinterpret_cast<__nv_bfloat16*>(out);
    a.fuse = fuse;
  }
  // Tile schedule of the CTA-pair kernels (AMOE_FFN_SCHED, read per launch):
  //   auto / dynamic (default): clusters claim the next raster unit from one atomic counter and
  //             hand it to the pair's roles through the shared-memory unit ring — the
  //             concurrently running units stay adjacent, so weight and token slabs are shared
  //             in L2 while hot (Mixtral gate/up DRAM reads 6.5-13 -> 3.1 GB per layer, tensor
  //             pipe 96.7 -> 98.4 % busy; DeepSeek down 78 -> 85 %)
  //   static  : cluster c takes units c, c + #clusters, ... of the raster
  //   die     : as dynamic, with each die owning its share of every queue's N tiles (needs a
  //             measured die split; otherwise dynamic)
  const char* ed = getenv("AMOE_FFN_SCHED");
  const int smode = !ed || !strcmp(ed, "auto") ? 3
                    : !strcmp(ed, "dynamic") ? 3 : !strcmp(ed, "die") ? (c.die_cnt[1] > 0 ? 1 : 3) : 0;
  a.die_sched = smode;
  // raster group: rows of a queue sharing a weight slab through L2. 4096 rows: the lowest DRAM
  // traffic measured for the static raster (gate/up 11.5 GB vs 15.5 GB at 2048 on a Mixtral layer,
  // profiles/r01_group_m_sweep.md); under the dynamic schedule the down GEMM (7 MB token slabs)
  // reads least with 2048-row groups (5.8-6.1 vs 8.3-8.5 GB, bench +0.8 %)
  const char* eg = getenv(part == 2 && getenv("AMOE_GROUP_M_DOWN") ? "AMOE_GROUP_M_DOWN" : "AMOE_GROUP_M");
  const int gm_rows = eg ? atoi(eg) : (part == 2 && pair && smode ? 2048 : 4096);
  a.group_m = std::max(1, gm_rows / (pair ? 256 : 128));
  if (pair) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(num_sms & ~1));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = tc2::SMEM2_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const int slots = (num_sms & ~1) / 2;
    if (part == 1) {
      cudaLaunchKernelEx(&cfg, tc2::ffn_tc2_kernel<MODE_GATEUP>, tm_tile, a, c);
      if (a.allow_split && reduce) launch_pdl(splitk_reduce_kernel<MODE_GATEUP, 256, true>, dim3(num_sms * 2), dim3(256), 0, s, a, c, slots);
    } else {
      cudaLaunchKernelEx(&cfg, tc2::ffn_tc2_kernel<MODE_DOWN>, tm_act, a, c);
      if (a.allow_split && reduce) launch_pdl(splitk_reduce_kernel<MODE_DOWN, 256, true>, dim3(num_sms * 2), dim3(256), 0, s, a, c, slots);
    }
    return a.allow_split && reduce ? 2 : 1;
  }
  if (part == 1) {
    launch_pdl(ffn_tc_kernel<MODE_GATEUP, 256>, dim3(num_sms), dim3(THREADS), SMEM_BYTES, s, tm_tile, tm_tile32, a, c);
    if (a.allow_split && reduce) launch_pdl(splitk_reduce_kernel<MODE_GATEUP, 256, false>, dim3(num_sms * 2), dim3(256), 0, s, a, c, num_sms);
  } else if (bn == 256) {
    launch_pdl(ffn_tc_kernel<MODE_DOWN, 256>, dim3(num_sms), dim3(THREADS), SMEM_BYTES, s, tm_act, tm_act32, a, c);
    if (a.allow_split && reduce) launch_pdl(splitk_reduce_kernel<MODE_DOWN, 256, false>, dim3(num_sms * 2), dim3(256), 0, s, a, c, num_sms);
  } else {
    launch_pdl(ffn_tc_kernel<MODE_DOWN, 128>, dim3(num_sms), dim3(THREADS), SMEM_BYTES, s, tm_act, tm_act32, a, c);
    if (a.allow_split && reduce) launch_pdl(splitk_reduce_kernel<MODE_DOWN, 128, false>, dim3(num_sms * 2), dim3(256), 0, s, a, c, num_sms);
  }
  return a.allow_split && reduce ? 2 : 1;
}

}  // namespace amoe
