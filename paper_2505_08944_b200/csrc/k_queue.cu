#include <stdlib.h>
// k_queue.cu — expert-side µ-queue kernels (owner rank):
//   drain   : a4 step 1 — take the published FIFO prefix of each selected µ-queue (PAPER.md
//             L222 "executor drains the selected queue"), allot 128-aligned rows per queue
//   gather  : a4 step 2 — the "custom CUDA kernel for preparing a contiguous input token batch
//             from many individually arrived token batches" (L222): pull each leg's x row from
//             its home (local load or NVLink peer load) into the contiguous tile
//   forward : a7 return leg — store each output row into the home's token pool (L236, one-sided
//             NVLink store replacing ZeroMQ+NCCL, L303-L320), bump the leg counter, and append
//             the token to its home's combine ring when its K (+S) legs are complete (L228)
#include "amoe_internal.cuh"

namespace amoe {

// AMOE_PDL=0 launches every kernel without programmatic dependent launch (A/B)
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("AMOE_PDL");
    on = e ? (e[0] != '0') : 1;
  }
  return on != 0;
}


constexpr int kDrainThreads = 128;

// Checked mode: append one record per nonempty drained queue and a copy of its drained legs
// (seq replaced by the token's pass, read from its home's token state) to the execution log.
// Called by every thread of the draining CTA after avail[]/head[] are final.
__device__ void xlog_drain(const DevCtx& c, int nq, const int32_t* qid, const uint32_t* head, const uint32_t* avail) {
  __shared__ uint32_t s_e0, s_l0;
  __shared__ uint32_t s_off[AMOE_MAX_GROUP];
  uint32_t* xl = c.xlog;
  if (threadIdx.x == 0) {
    uint32_t ne = 0, nl = 0;
    for (int q = 0; q < nq; ++q)
      if (avail[q]) { s_off[q] = nl; nl += avail[q]; ++ne; }
    s_e0 = atomicAdd(xl + 0, ne);
    s_l0 = atomicAdd(xl + 1, nl);
    uint32_t e = s_e0;
    for (int q = 0; q < nq; ++q)
      if (avail[q]) {
        if (e < xl[2]) {
          uint32_t* r = xlog_exec(xl) + 4 * (uint64_t)e;
          r[0] = (uint32_t)qid[q]; r[1] = head[q]; r[2] = avail[q]; r[3] = s_l0 + s_off[q];
        }
        ++e;
      }
  }
  __syncthreads();
  amoe_leg* legs = xlog_legs(xl);
  const uint32_t cap = xl[3];
  for (int q = 0; q < nq; ++q) {
    if (!avail[q]) continue;
    const amoe_leg* ring = ring_ptr(c, c.rank, qid[q]);
    for (uint32_t i = threadIdx.x; i < avail[q]; i += blockDim.x) {
      const uint32_t o = s_l0 + s_off[q] + i;
      if (o >= cap) break;
      amoe_leg e = ring[(head[q] + i) & c.ring_mask];
      const int home = (e.home >= 0 && e.home < c.G) ? e.home : c.rank;
      const int slot = (e.token_slot >= 0 && e.token_slot < c.T) ? e.token_slot : 0;
      e.seq = (uint32_t)reinterpret_cast<const int32_t*>(c.peer[home] + c.lay.tok_pass)[slot];
      legs[o] = e;
    }
  }
}

__global__ void __launch_bounds__(kDrainThreads) drain_kernel(DevCtx c, GroupDev g) {
  AMOE_PDL_ENTRY();
  __shared__ uint32_t avail[AMOE_MAX_GROUP], head[AMOE_MAX_GROUP], rv[AMOE_MAX_GROUP];
  __shared__ int slow[AMOE_MAX_GROUP];
  __shared__ int nslow;
  const int tid = threadIdx.x;
  if (tid == 0) nslow = 0;
  __syncthreads();
  for (int q = tid; q < g.nq; q += blockDim.x) {
    uint32_t* ctr = qctr_ptr(c, c.rank, g.qid[q]);
    const uint32_t cm = ld_acquire(ctr + 1);
    const uint32_t r = ld_relaxed(ctr + 0);
    head[q] = ctr[2];
    rv[q] = r;
    if (r - head[q] > c.ring_cap) raise_fault(c, F_RING_OVERFLOW, g.qid[q], r, head[q]);
    if (g.exact) {
      // the scheduler's count (<= the published count it saw): taken whole. When no producer is
      // mid-flight (commit == reserve) the acquire on commit already covers every entry below it;
      // otherwise the entries of [head, head + cap) are waited for below
      avail[q] = (uint32_t)g.cap[q];
      if (!(cm == r && avail[q] <= cm - head[q])) slow[atomicAdd(&nslow, 1)] = q;
    } else if (cm == r) {
      avail[q] = cm - head[q];
    } else {
      avail[q] = 0;
      slow[atomicAdd(&nslow, 1)] = q;
    }
  }
  __syncthreads();
  if (g.exact) {
    for (int sq = 0; sq < nslow; ++sq) {
      const int q = slow[sq];
      const amoe_leg* ring = ring_ptr(c, c.rank, g.qid[q]);
      for (uint32_t i = tid; i < avail[q]; i += blockDim.x) {
        const uint32_t pos = head[q] + i;
        if (ld_acquire(&ring[pos & c.ring_mask].seq) != pos + 1u) {
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire(&ring[pos & c.ring_mask].seq) != pos + 1u)
            if (globaltimer_ns() - t0 > 4000000000ull) { raise_fault(c, F_STALE_ENTRY, g.qid[q], pos, 0); break; }
        }
      }
    }
    __syncthreads();
    if (tid == 0) nslow = 0;
    __syncthreads();
  }
  // slow path: a producer on a peer is mid-flight; the published prefix is where seq == pos+1
  for (int s = 0; s < nslow; ++s) {
    const int q = slow[s];
    const amoe_leg* ring = ring_ptr(c, c.rank, g.qid[q]);
    __shared__ int stop;
    uint32_t n = 0;
    for (;;) {
      const uint32_t pos = head[q] + n + tid;
      const bool ok = (pos - head[q]) < (rv[q] - head[q]) &&
                      ld_acquire(&ring[pos & c.ring_mask].seq) == pos + 1u;
      if (tid == 0) stop = blockDim.x;
      __syncthreads();
      if (!ok) atomicMin(&stop, tid);
      __syncthreads();
      const int st = stop;
      __syncthreads();
      if (st < (int)blockDim.x) { n += st; break; }
      n += blockDim.x;
    }
    if (tid == 0) avail[q] = n;
    __syncthreads();
  }
  if (tid == 0) {
    uint32_t off = 0;
    for (int q = 0; q < g.nq; ++q) {
      uint32_t n = avail[q];
      if (g.max_tokens > 0 && n > (uint32_t)g.max_tokens) n = g.max_tokens;
      const uint32_t room = off < (uint32_t)g.rows_cap ? (uint32_t)g.rows_cap - off : 0u;
      if (n > room) n = room;
      g.qinfo[q] = (int32_t)n;
      g.qinfo[AMOE_MAX_GROUP + q] = (int32_t)off;
      g.qinfo[2 * AMOE_MAX_GROUP + q] = (int32_t)head[q];
      avail[q] = n;
      off += (n + kRowAlign - 1) / kRowAlign * kRowAlign;
    }
  }
  __syncthreads();
  for (int q = tid; q < g.nq; q += blockDim.x) qctr_ptr(c, c.rank, g.qid[q])[2] = head[q] + avail[q];
  if (c.xlog) xlog_drain(c, g.nq, g.qid, head, avail);
}

// Locate the queue of row-rank r in a group (prefix sums of n in shared memory).
__device__ __forceinline__ int find_queue(const int* pre, int nq, int r) {
  int lo = 0, hi = nq - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

constexpr int kRowThreads = 256;

__global__ void __launch_bounds__(kRowThreads) gather_kernel(DevCtx c, GroupDev g) {
  AMOE_PDL_ENTRY();
  __shared__ int pre[AMOE_MAX_GROUP + 1];
  __shared__ int n_s[AMOE_MAX_GROUP], off_s[AMOE_MAX_GROUP], start_s[AMOE_MAX_GROUP];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < g.nq; ++q) {
      n_s[q] = g.qinfo[q]; off_s[q] = g.qinfo[AMOE_MAX_GROUP + q]; start_s[q] = g.qinfo[2 * AMOE_MAX_GROUP + q];
      pre[q] = acc; acc += n_s[q];
    }
    pre[g.nq] = acc;
  }
  __syncthreads();
  const int total = pre[g.nq];
  const int lane = threadIdx.x & 31;
  const int rowbytes = c.d * c.esize;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < total; r += nw) {
    const int q = find_queue(pre, g.nq, r);
    const int i = r - pre[q];
    const uint32_t pos = (uint32_t)start_s[q] + (uint32_t)i;
    const amoe_leg e = ring_ptr(c, c.rank, g.qid[q])[pos & c.ring_mask];
    const int row = off_s[q] + i;
    if (e.seq != pos + 1u || e.home < 0 || e.home >= c.G || e.token_slot < 0 || e.token_slot >= c.T) {
      if (lane == 0) raise_fault(c, F_STALE_ENTRY, g.qid[q], pos, e.seq);
      continue;
    }
    if (lane == 0) g.meta[row] = e;
    const char* src = reinterpret_cast<const char*>(c.peer[e.home] + c.lay.x) + (uint64_t)e.token_slot * rowbytes;
    char* dst = reinterpret_cast<char*>(g.tile) + (uint64_t)row * rowbytes;
    warp_copy(dst, src, rowbytes, lane);
  }
}

__global__ void __launch_bounds__(kRowThreads) forward_kernel(DevCtx c, GroupDev g) {
  AMOE_PDL_ENTRY();
  __shared__ int pre[AMOE_MAX_GROUP + 1];
  __shared__ int off_s[AMOE_MAX_GROUP];
  __shared__ unsigned long long s_legs, s_remote;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < g.nq; ++q) { off_s[q] = g.qinfo[AMOE_MAX_GROUP + q]; pre[q] = acc; acc += g.qinfo[q]; }
    pre[g.nq] = acc;
    s_legs = 0; s_remote = 0;
  }
  __syncthreads();
  const int total = pre[g.nq];
  const int lane = threadIdx.x & 31;
  const int rowbytes = c.d * c.esize;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < total; r += nw) {
    const int q = find_queue(pre, g.nq, r);
    const int row = off_s[q] + (r - pre[q]);
    const amoe_leg e = g.meta[row];
    const int home = e.home;
    const bool sys = c.G > 1;            // all writers of a leg counter use one scope
    char* dst = reinterpret_cast<char*>(c.peer[home] + c.lay.pool) +
                ((uint64_t)e.token_slot * c.KS + (uint64_t)e.k) * rowbytes;
    const char* src = reinterpret_cast<const char*>(g.out) + (uint64_t)row * rowbytes;
    warp_copy(dst, src, rowbytes, lane);
    __syncwarp();
    if (lane == 0) {
      fence_sc(sys);       // the whole warp's row stores before the counter (cumulativity)
      atomicAdd(&s_legs, 1ull);
      if (home != c.rank) atomicAdd(&s_remote, 1ull);
      // the whole row = d columns; the completing arrival appends to the combine ring
      leg_pieces_done(c, home, e.token_slot, e.k, (uint32_t)c.d);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* st = wsp<unsigned long long>(c, c.rank, c.lay.stats);
    if (s_legs) atomicAdd(st + 2, s_legs);
    if (s_remote) atomicAdd(st + 3, s_remote);
  }
}

// AMOE_DEFRAG_GLOBAL: box-wide queued legs per block, read from every
// rank's queue counters (peer loads over NVLink; the counters are the same published-minus-
// drained depths each rank's own scheduler snapshots) into this rank's gtot[L], which the next
// host snapshot copies. One CTA per block.
__global__ void peer_depths_kernel(DevCtx c) {
  AMOE_PDL_ENTRY();
  const int b = blockIdx.x;
  uint32_t tot = 0;
  for (int i = threadIdx.x; i < c.G * c.H; i += blockDim.x) {
    const int r = i / c.H, q = i - r * c.H;
    const uint32_t* qc = qctr_ptr(c, r, b * c.H + q);
    tot += ld_relaxed(qc + 1) - ld_relaxed(qc + 2);
  }
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  __shared__ uint32_t s_tot[kRowThreads / 32];
  if ((threadIdx.x & 31) == 0) s_tot[threadIdx.x >> 5] = tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_tot[w];
    wsp<uint32_t>(c, c.rank, c.lay.gtot)[b] = t;
  }
}

int launch_peer_depths(const DevCtx& c, cudaStream_t s) {
  launch_pdl(peer_depths_kernel, dim3(c.L), dim3(kRowThreads), 0, s, c);
  return 1;
}

int launch_drain(const DevCtx& c, const GroupDev& g, cudaStream_t s) {
  launch_pdl(drain_kernel, dim3(1), dim3(kDrainThreads), 0, s, c, g);
  return 1;
}

static int row_grid(const DevCtx& c, int num_sms) {
  // enough warps to cover the worst-case rows, capped at 8 CTAs per SM
  (void)c;
  return num_sms * 8;
}

int launch_gather(const DevCtx& c, const GroupDev& g, int num_sms, cudaStream_t s) {
  launch_pdl(gather_kernel, dim3(row_grid(c, num_sms)), dim3(kRowThreads), 0, s, c, g);
  return 1;
}

int launch_forward(const DevCtx& c, const GroupDev& g, int num_sms, cudaStream_t s) {
  launch_pdl(forward_kernel, dim3(row_grid(c, num_sms)), dim3(kRowThreads), 0, s, c, g);
  return 1;
}

}  // namespace amoe
