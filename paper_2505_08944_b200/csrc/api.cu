// api.cu — host side of libamoe: the C ABI of include/amoe.h, the workspace layout, TMA
// descriptor encoding, and the asynchronous scheduler loop (amoe_run).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <vector>

#include "amoe_internal.cuh"

namespace amoe {
// kernels (k_*.cu)
int launch_token_init(const DevCtx&, const int32_t*, int, const void*, int, cudaStream_t);
int launch_enqueue(const DevCtx&, int, const int32_t*, int, const float*, const int32_t*, const float*, cudaStream_t);
int launch_combine(const DevCtx&, int, int, cudaStream_t);
int launch_announce(const DevCtx&, uint32_t, int, cudaStream_t);
int launch_direct_merge(const DevCtx&, const GroupDev&, int, int, cudaStream_t);
int die_map(uint64_t mask[4], int counts[2]);
int launch_drain(const DevCtx&, const GroupDev&, cudaStream_t);
int launch_gather(const DevCtx&, const GroupDev&, int, cudaStream_t);
int launch_forward(const DevCtx&, const GroupDev&, int, cudaStream_t);
int launch_ffn_tc(const DevCtx&, const FfnLaunch&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                  const CUtensorMap&, void*, void*, const amoe_leg*, int, int, int, cudaStream_t, int);
int launch_ffn_cold(const DevCtx&, int, const int*, const int*, const uint32_t*, int, int, int, const CUtensorMap&, void*,
                    int32_t*, const CUtensorMap*, const CUtensorMap*, int, cudaStream_t);
void cold_blocks(int d, int ff, int n_pad, int* ka, int* kb);
int launch_ffn_simt(const DevCtx&, int, const int32_t*, const int*, const uint64_t*, const void*, void*, void*, int, cudaStream_t);
int pick_queue(const uint32_t* Q, int NB, int H, int NE, int policy, int W, double delta, int* b, int* q,
               const uint32_t* look = nullptr);
int launch_peer_depths(const DevCtx&, cudaStream_t);
}  // namespace amoe

using namespace amoe;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct MapCacheEntry {
  const void* ptr;
  int rows, cols, box_rows, depth;
  CUtensorMap map;
};

struct amoe_ctx {
  amoe_config cfg;
  bool direct = false;                // top-1 direct forwarding (amoe_set_direct)
  uint64_t merged_seen = 0;           // home merge counter at the end of the last amoe_run
  const int32_t* exact_caps = nullptr;  // set by amoe_run's pipelined loop around a pick's launches
  uint32_t* snapbuf[3] = {nullptr, nullptr, nullptr};   // pipelined loop: rotating pinned snapshots
  cudaEvent_t snapev[6] = {};          // [b]: copy b landed; [3 + b]: compute stream reached copy b
  cudaStream_t copy_stream = nullptr;  // the snapshot copies' side stream
  DevCtx dc;
  Layout lay;
  char* ws;
  size_t ws_bytes;
  int num_sms;
  int Hr, H;
  std::vector<int> hosted_flags;      // [L*H] weights registered
  std::vector<uint64_t> wptrs;        // [L*H*3]
  uint32_t* pinned;                   // snapshot buffer (header + qctr)
  size_t snap_bytes;
  int64_t launches;
  int64_t admitted;
  uint64_t retired_base;
  uint32_t epoch;
  std::vector<char> gate_set;         // [L] layer has a router gate (amoe_set_gate)
  int start_layer = 0;                // layer of the last amoe_enqueue (AMOE_SYNC's first layer)
  cudaStream_t last_stream;
  std::vector<MapCacheEntry> map_cache;
  int32_t* scratch_qinfo;
  // per-stage device timing (amoe_profile_*): CUDA events bracket each stage on its stream
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  double prof_ms[8] = {0};
  int64_t prof_n[8] = {0};
  // executions logged by amoe_run while profiling: (l*H + q, drained legs), from the ring heads
  std::vector<uint32_t> prev_head;
  std::vector<int32_t> exec_log;
};

enum Stage { ST_REBATCH = 0, ST_GATEUP = 1, ST_DOWN = 2, ST_FORWARD = 3, ST_COMBINE = 4, ST_ENQUEUE = 5, ST_COLD = 6 };

static cudaEvent_t ev_get(amoe_ctx* c) {
  if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct StageTimer {
  amoe_ctx* c; int stage; cudaStream_t s; cudaEvent_t a = nullptr;
  StageTimer(amoe_ctx* c_, int st, cudaStream_t s_) : c(c_), stage(st), s(s_) {
    if (c->prof) { a = ev_get(c); cudaEventRecord(a, s); }
  }
  ~StageTimer() {
    if (c->prof) { cudaEvent_t b = ev_get(c); cudaEventRecord(b, s); c->recs.push_back({stage, a, b}); }
  }
};

static PFN_encodeTiled get_encoder() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// 2D bf16 row-major matrix [rows, cols] -> TMA map with a {64, box_rows} box, 128-B swizzle.
static bool encode_bf16_2d(CUtensorMap* m, const void* ptr, int rows, int cols, int box_rows) {
  PFN_encodeTiled enc = get_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// The same matrix seen as `depth`-deep stacks of K blocks: dims {64, rows, cols/64}, strides
// {cols*2, 128 B}, box {64, box_rows, depth}. One load lands as `depth` consecutive K-major
// 128-B-swizzled tiles [kb][box_rows][64] (tools/tma3d_probe.cu checks the layout), so a ring
// stage needs one TMA box per operand instead of one per K block: a B200 SM retires a roughly
// fixed number of boxes per microsecond whatever their size up to 32 KB (tools/tma_stream_probe.cu).
static bool encode_bf16_kb3d(CUtensorMap* m, const void* ptr, int rows, int cols, int box_rows, int depth) {
  PFN_encodeTiled enc = get_encoder();
  if (!enc || cols % (64 * depth)) return false;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)depth};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// depth 0: the 2-D map; > 0: the K-block view of that depth
static const CUtensorMap* cached_map(amoe_ctx* c, const void* ptr, int rows, int cols, int box_rows, int depth = 0) {
  for (auto& e : c->map_cache)
    if (e.ptr == ptr && e.rows == rows && e.cols == cols && e.box_rows == box_rows && e.depth == depth) return &e.map;
  MapCacheEntry e{ptr, rows, cols, box_rows, depth, {}};
  if (depth == 0 ? !encode_bf16_2d(&e.map, ptr, rows, cols, box_rows)
                 : !encode_bf16_kb3d(&e.map, ptr, rows, cols, box_rows, depth))
    return nullptr;
  if (c->map_cache.size() > 64) c->map_cache.erase(c->map_cache.begin());
  c->map_cache.push_back(e);
  return &c->map_cache.back().map;
}

static uint32_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return (uint32_t)p;
}

static inline uint64_t al(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

static bool valid_cfg(const amoe_config* c) {
  if (!c) return false;
  if (c->L < 1 || c->E < 1 || c->E > AMOE_MAX_E || c->K < 1 || c->K > 8 || c->K > c->E) return false;
  if (c->S < 0 || c->S > 4 || c->K + c->S > kMaxKS) return false;
  if (c->d < 128 || c->d % 128 || c->ff < 128 || c->ff % 128) return false;
  if (c->G < 1 || c->G > AMOE_MAX_G || c->rank < 0 || c->rank >= c->G) return false;
  if (c->T_slots < 1 || c->dtype < 0 || c->dtype > 1 || c->max_batch < 0 || c->rows_cap < 0) return false;
  for (int e = 0; e < c->E; ++e)
    if (c->owner[e] < 0 || c->owner[e] >= c->G) return false;
  return true;
}

// owner table: all-zero with G > 1 means the default e mod G
static void resolve_owner(const amoe_config* c, int* owner) {
  bool allzero = true;
  for (int e = 0; e < c->E; ++e) allzero &= c->owner[e] == 0;
  for (int e = 0; e < c->E; ++e) owner[e] = (allzero && c->G > 1) ? e % c->G : c->owner[e];
}

static void compute_layout(const amoe_config* c, Layout* L, int* Hr_out, uint32_t* ring_cap, uint32_t* cring_cap) {
  int owner[AMOE_MAX_E];
  resolve_owner(c, owner);
  int cnt[AMOE_MAX_G] = {0};
  for (int e = 0; e < c->E; ++e) cnt[owner[e]]++;
  int Hr = 0;
  for (int r = 0; r < c->G; ++r) Hr = std::max(Hr, cnt[r]);
  const int H = Hr + c->S;
  const uint64_t es = c->dtype == AMOE_BF16 ? 2 : 4;
  const uint64_t T = c->T_slots, d = c->d, ff = c->ff, KS = c->K + c->S;
  const uint32_t rc = next_pow2(std::max<uint64_t>((uint64_t)c->G * T, 2));
  const uint32_t crc = next_pow2(std::max<uint64_t>(T, 2));
  int rows = c->rows_cap;
  if (rows == 0) {
    const uint64_t legs = (uint64_t)c->G * T * (uint64_t)std::min(c->K, std::max(Hr, 1)) + T * c->S;
    rows = (int)std::min<uint64_t>(legs + (uint64_t)H * kRowAlign, 0x7fffffff);
  }
  rows = (int)al((uint64_t)rows, kRowAlign);
  uint64_t o = 0;
  auto take = [&](uint64_t bytes, uint64_t a = 256) { o = al(o, a); uint64_t r = o; o += bytes; return r; };
  L->err = take(64);
  L->stats = take(64, 64);
  L->done = take(64, 64);
  L->cctr = take(64, 64);
  L->gtot = take((uint64_t)c->L * 4, 64);
  L->qctr = take((uint64_t)c->L * H * 16, 64);     // snapshot = [0, qctr end)
  L->rings = take((uint64_t)c->L * H * rc * 16);
  L->cring = take((uint64_t)crc * 16);
  L->cinfo = take(16);
  L->sched = take(16);
  L->split_cnt = take((uint64_t)kSplitSlots * 4);
  L->cold = take((uint64_t)kColdCtr * 4);
  L->h = take(T * d * es);
  L->x = take(T * d * es);
  L->pool = take(T * KS * d * es);
  L->legs_done = take(T * 4);
  L->tok_layer = take(T * 4);
  L->tok_pass = take(T * 4);
  L->tok_w = take(T * c->K * 4);
  L->tok_idx = take(T * c->K * 4);
  L->tok_time = take(T * 16, 16);
  L->wmaps = take((uint64_t)c->L * H * 3 * 128, 128);
  L->cmaps = take((uint64_t)c->L * H * 4 * 128, 128);
  L->wptrs = take((uint64_t)c->L * H * 3 * 8);
  L->gate = take((uint64_t)c->L * 16);
  L->s_qinfo = take(3 * AMOE_MAX_GROUP * 4);
  L->s_meta = take((uint64_t)rows * 16);
  L->s_tile = take((uint64_t)rows * d * es, 1024);
  L->s_act = take((uint64_t)rows * ff * es, 1024);
  L->s_out = take((uint64_t)rows * d * es, 1024);
  L->split_part = take((uint64_t)kSplitUnits * 128 * 256 * 4, 1024);
  L->total = al(o, 256);
  L->rows_cap = rows;
  *Hr_out = Hr;
  *ring_cap = rc;
  *cring_cap = crc;
}

#define CK(x)                                   \
  do {                                          \
    if ((x) != cudaSuccess) return AMOE_ECUDA;  \
  } while (0)

extern "C" {

size_t amoe_workspace_bytes(const amoe_config* cfg) {
  if (!valid_cfg(cfg)) return 0;
  Layout L;
  int Hr;
  uint32_t rc, crc;
  compute_layout(cfg, &L, &Hr, &rc, &crc);
  return (size_t)L.total;
}

const char* amoe_status_string(amoe_status s) {
  switch (s) {
    case AMOE_OK: return "ok";
    case AMOE_IDLE: return "idle: all hosted queues empty";
    case AMOE_EINVAL: return "invalid argument";
    case AMOE_ENOTHOSTED: return "expert not hosted on this rank";
    case AMOE_ECUDA: return "CUDA runtime error";
    case AMOE_EDEVICE: return "device-side invariant breach (see amoe_error_info)";
    case AMOE_EPEER: return "peer workspaces missing or inconsistent";
    case AMOE_ENOMEM: return "workspace too small";
  }
  return "unknown status";
}

amoe_status amoe_create(const amoe_config* cfg, void* workspace, size_t bytes, amoe_ctx_t* out) {
  if (!valid_cfg(cfg) || !workspace || !out || (reinterpret_cast<uintptr_t>(workspace) & 255)) return AMOE_EINVAL;
  amoe_ctx* c = new amoe_ctx();
  c->cfg = *cfg;
  uint32_t rc, crc;
  compute_layout(cfg, &c->lay, &c->Hr, &rc, &crc);
  if (bytes < c->lay.total) { delete c; return AMOE_ENOMEM; }
  c->H = c->Hr + cfg->S;
  c->ws = static_cast<char*>(workspace);
  c->ws_bytes = bytes;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  // AMOE_NUM_SMS: persistent grids of this context sized for fewer SMs (contexts of one process
  // co-running on disjoint halves of a GPU emulate G GPUs: tools/g_emulate.py)
  if (const char* e = getenv("AMOE_NUM_SMS")) {
    const int n = atoi(e);
    if (n >= 2 && n < c->num_sms) c->num_sms = n & ~1;
  }
  DevCtx& d = c->dc;
  memset(&d, 0, sizeof(d));
  d.L = cfg->L; d.E = cfg->E; d.K = cfg->K; d.S = cfg->S; d.d = cfg->d; d.ff = cfg->ff;
  d.G = cfg->G; d.rank = cfg->rank; d.T = cfg->T_slots; d.dtype = cfg->dtype;
  d.H = c->H; d.Hr = c->Hr; d.KS = cfg->K + cfg->S; d.esize = cfg->dtype == AMOE_BF16 ? 2 : 4;
  d.ring_cap = rc; d.ring_mask = rc - 1; d.cring_cap = crc; d.cring_mask = crc - 1;
  d.eps = cfg->rms_eps > 0.f ? cfg->rms_eps : 1e-6f;
  d.n_tab = 0; d.router = nullptr;
  die_map(d.die_mask, d.die_cnt);     // cached per device after the first context
  d.lay = c->lay;
  int owner[AMOE_MAX_E];
  resolve_owner(cfg, owner);
  int cnt[AMOE_MAX_G] = {0};
  for (int e = 0; e < cfg->E; ++e) { d.owner[e] = (uint8_t)owner[e]; d.lq[e] = (int16_t)cnt[owner[e]]++; }
  for (int r = 0; r < AMOE_MAX_G; ++r) d.peer[r] = 0;
  d.peer[cfg->rank] = reinterpret_cast<uint64_t>(workspace);
  c->hosted_flags.assign((size_t)cfg->L * c->H, 0);
  c->wptrs.assign((size_t)cfg->L * c->H * 3, 0);
  c->snap_bytes = c->lay.qctr + (uint64_t)cfg->L * c->H * 16;
  if (cudaMallocHost(&c->pinned, c->snap_bytes) != cudaSuccess) { delete c; return AMOE_ECUDA; }
  // zero counters, rings (seq flags) and token state; h/x/pool/scratch tiles need no init
  if (cudaMemset(c->ws, 0, c->lay.h) != cudaSuccess ||
      cudaMemset(c->ws + c->lay.legs_done, 0, c->lay.wmaps - c->lay.legs_done) != cudaSuccess ||
      cudaMemset(c->ws + c->lay.wptrs, 0, c->lay.s_meta - c->lay.wptrs) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaFreeHost(c->pinned);
    delete c;
    return AMOE_ECUDA;
  }
  c->launches = 0; c->admitted = 0; c->retired_base = 0; c->epoch = 0;
  c->last_stream = 0;
  *out = c;
  return AMOE_OK;
}

amoe_status amoe_import_peers(amoe_ctx_t c, const uint64_t* peer_ws, int G) {
  if (!c || !peer_ws || G != c->cfg.G) return AMOE_EINVAL;
  if (peer_ws[c->cfg.rank] != reinterpret_cast<uint64_t>(c->ws)) return AMOE_EPEER;
  for (int r = 0; r < G; ++r)
    if (!peer_ws[r] || (peer_ws[r] & 255)) return AMOE_EPEER;
  // kernels of this device dereference every peer workspace (one-sided legs over NVLink): a
  // workspace that lives on another device needs peer access from this one. An IPC handle
  // opened under the peer's device guard does not grant it, so enable it here (idempotent).
  int me = -1;
  CK(cudaGetDevice(&me));
  for (int r = 0; r < G; ++r) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, reinterpret_cast<const void*>(peer_ws[r])) != cudaSuccess) {
      cudaGetLastError();
      return AMOE_EPEER;              // not a device address in this process
    }
    if (a.type == cudaMemoryTypeDevice && a.device >= 0 && a.device != me) {
      int can = 0;
      CK(cudaDeviceCanAccessPeer(&can, me, a.device));
      if (!can) return AMOE_EPEER;
      const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return AMOE_ECUDA;
    }
  }
  for (int r = 0; r < G; ++r) c->dc.peer[r] = peer_ws[r];
  return AMOE_OK;
}

int amoe_hosted(amoe_ctx_t c) { return c ? c->H : -1; }
int amoe_ring_cap(amoe_ctx_t c) { return c ? (int)c->dc.ring_cap : -1; }
int amoe_local_queue(amoe_ctx_t c, int e) {
  if (!c || e < 0) return -1;
  if (e < c->cfg.E) return c->dc.lq[e];
  if (e < c->cfg.E + c->cfg.S) return c->Hr + (e - c->cfg.E);
  return -1;
}
int64_t amoe_launch_count(amoe_ctx_t c) { return c ? c->launches : -1; }

// queue slot (l*H + local) of (layer, expert) on THIS rank, or -1 if not hosted
static int local_slot(amoe_ctx* c, int layer, int expert) {
  if (layer < 0 || layer >= c->cfg.L) return -1;
  if (expert >= 0 && expert < c->cfg.E) {
    if (c->dc.owner[expert] != c->cfg.rank) return -1;
    return layer * c->H + c->dc.lq[expert];
  }
  if (expert >= c->cfg.E && expert < c->cfg.E + c->cfg.S) return layer * c->H + c->Hr + (expert - c->cfg.E);
  return -1;
}

amoe_status amoe_set_expert(amoe_ctx_t c, int layer, int expert, const void* w1, const void* w3, const void* w2) {
  if (!c || !w1 || !w3 || !w2) return AMOE_EINVAL;
  if (layer < 0 || layer >= c->cfg.L || expert < 0 || expert >= c->cfg.E + c->cfg.S) return AMOE_EINVAL;
  const int slot = local_slot(c, layer, expert);
  if (slot < 0) return AMOE_ENOTHOSTED;
  for (const void* p : {w1, w3, w2})
    if (reinterpret_cast<uintptr_t>(p) & 15) return AMOE_EINVAL;
  uint64_t ptrs[3] = {reinterpret_cast<uint64_t>(w1), reinterpret_cast<uint64_t>(w3), reinterpret_cast<uint64_t>(w2)};
  CK(cudaMemcpy(c->ws + c->lay.wptrs + (uint64_t)slot * 24, ptrs, 24, cudaMemcpyHostToDevice));
  if (c->cfg.dtype == AMOE_BF16) {
    CUtensorMap maps[3];
    if (!encode_bf16_2d(&maps[0], w1, c->cfg.ff, c->cfg.d, 128) ||
        !encode_bf16_2d(&maps[1], w3, c->cfg.ff, c->cfg.d, 128) ||
        !encode_bf16_2d(&maps[2], w2, c->cfg.d, c->cfg.ff, 128))
      return AMOE_ECUDA;
    CK(cudaMemcpy(c->ws + c->lay.wmaps + (uint64_t)slot * 3 * 128, maps, sizeof(maps), cudaMemcpyHostToDevice));
    // K-block views for the cold kernel: W1 / W3 two K blocks deep (128 rows), W2 two and one
    // deep over 256-row tiles (a view whose depth does not divide K stays zero, never selected)
    CUtensorMap cm[4];
    memset(cm, 0, sizeof(cm));
    encode_bf16_kb3d(&cm[0], w1, c->cfg.ff, c->cfg.d, 128, 2);
    encode_bf16_kb3d(&cm[1], w3, c->cfg.ff, c->cfg.d, 128, 2);
    encode_bf16_kb3d(&cm[2], w2, c->cfg.d, c->cfg.ff, 256, 2);   // down: 256-row tiles (§5.4)
    encode_bf16_kb3d(&cm[3], w2, c->cfg.d, c->cfg.ff, 256, 1);
    CK(cudaMemcpy(c->ws + c->lay.cmaps + (uint64_t)slot * 4 * 128, cm, sizeof(cm), cudaMemcpyHostToDevice));
  }
  for (int i = 0; i < 3; ++i) c->wptrs[(size_t)slot * 3 + i] = ptrs[i];
  c->hosted_flags[slot] = 1;
  return AMOE_OK;
}

amoe_status amoe_set_gate(amoe_ctx_t c, int layer, const void* wg, const float* bias) {
  if (!c || layer < 0 || layer >= c->cfg.L) return AMOE_EINVAL;
  // the gate keeps the token's x row in registers: 16 chunks of 16 B per lane
  if (wg && c->cfg.d > 16 * 32 * (16 / (int)c->dc.esize)) return AMOE_EINVAL;
  const uint64_t v[2] = {reinterpret_cast<uint64_t>(wg), wg ? reinterpret_cast<uint64_t>(bias) : 0};
  CK(cudaMemcpy(c->ws + c->lay.gate + (uint64_t)layer * 16, v, 16, cudaMemcpyHostToDevice));
  c->gate_set.resize(c->cfg.L, 0);
  c->gate_set[layer] = wg != nullptr;
  c->dc.gate_on = 0;
  for (char g : c->gate_set) c->dc.gate_on |= g;
  return AMOE_OK;
}

amoe_status amoe_set_direct(amoe_ctx_t c, int on) {
  if (!c) return AMOE_EINVAL;
  if (on && (c->cfg.K != 1 || c->cfg.S != 0)) return AMOE_EINVAL;
  c->direct = on != 0;
  return AMOE_OK;
}

amoe_status amoe_set_exec_log(amoe_ctx_t c, void* buf, size_t bytes) {
  if (!c) return AMOE_EINVAL;
  if (!buf) { c->dc.xlog = nullptr; return AMOE_OK; }
  if ((reinterpret_cast<uintptr_t>(buf) & 15) || bytes < (kXlogHeader + 4) * 4 + 16) return AMOE_EINVAL;
  // split the buffer: one 16-B exec record per 16 drained legs (an execution drains >= 1 leg)
  const uint64_t body = bytes - kXlogHeader * 4;
  uint64_t cap_e = body / 16 / 8;
  if (cap_e < 1) cap_e = 1;
  const uint64_t cap_l = (body - cap_e * 16) / 16;
  if (cap_l < 1 || cap_e > 0xffffffffu || cap_l > 0xffffffffu) return AMOE_EINVAL;
  const uint32_t hdr[kXlogHeader] = {0, 0, (uint32_t)cap_e, (uint32_t)cap_l, 0, 0, 0, 0};
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(buf, hdr, sizeof(hdr), cudaMemcpyHostToDevice));
  c->dc.xlog = static_cast<uint32_t*>(buf);
  return AMOE_OK;
}

amoe_status amoe_set_router(amoe_ctx_t c, const float* table, int n_tables) {
  if (!c || !table || n_tables < 1) return AMOE_EINVAL;
  c->dc.router = table;
  c->dc.n_tab = n_tables;
  return AMOE_OK;
}

amoe_status amoe_token_init(amoe_ctx_t c, const int32_t* slots, int T, const void* h0, int pass, void* stream) {
  if (!c || T < 0 || (T > 0 && (!slots || !h0))) return AMOE_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  StageTimer tm(c, ST_ENQUEUE, s);
  c->launches += launch_token_init(c->dc, slots, T, h0, pass, s);
  c->admitted += T;
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

amoe_status amoe_enqueue(amoe_ctx_t c, int layer, const int32_t* slots, int T, const float* logits,
                         const int32_t* topk_idx, const float* topk_w, void* stream) {
  if (!c || T < 0 || layer < 0 || layer >= c->cfg.L) return AMOE_EINVAL;
  // no logits and no (idx, w): route with the layer's gate (amoe_set_gate) on the tokens' x
  if (T > 0 && (!slots || (!logits && (!topk_idx || !topk_w) && !c->dc.gate_on))) return AMOE_EINVAL;
  if (!logits && (!topk_idx || !topk_w)) { topk_idx = nullptr; topk_w = nullptr; }
  cudaStream_t s = (cudaStream_t)stream;
  for (int r = 0; r < c->cfg.G; ++r)
    if (!c->dc.peer[r]) return AMOE_EPEER;
  StageTimer tm(c, ST_ENQUEUE, s);
  c->launches += launch_enqueue(c->dc, layer, slots, T, logits, topk_idx, topk_w, s);
  c->start_layer = layer;
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

static amoe_status snapshot(amoe_ctx* c, cudaStream_t s) {
  CK(cudaMemcpyAsync(c->pinned, c->ws, c->snap_bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AMOE_OK;
}

// Executions since the previous snapshot: a queue's consumer head only moves when a pick drains
// it, and one poll launches at most one pick (each queue at most once), so every head delta
// between consecutive snapshots is exactly one execution of that many legs.
static void log_executions(amoe_ctx* c, bool reset) {
  const uint32_t* q = c->pinned + c->lay.qctr / 4;
  const int n = c->cfg.L * c->H;
  c->prev_head.resize(n);
  for (int i = 0; i < n; ++i) {
    const uint32_t h = q[4 * i + 2];
    if (!reset && c->prof && h != c->prev_head[i]) {
      c->exec_log.push_back(i);
      c->exec_log.push_back((int32_t)(h - c->prev_head[i]));
    }
    c->prev_head[i] = h;
  }
}

static void depths_from_snapshot(amoe_ctx* c, uint32_t* Q) {
  const uint32_t* q = c->pinned + c->lay.qctr / 4;
  const int n = c->cfg.L * c->H;
  for (int i = 0; i < n; ++i) Q[i] = q[4 * i + 1] - q[4 * i + 2];
}

amoe_status amoe_queue_depths(amoe_ctx_t c, uint32_t* host_out, void* stream) {
  if (!c || !host_out) return AMOE_EINVAL;
  amoe_status st = snapshot(c, (cudaStream_t)stream);
  if (st != AMOE_OK) return st;
  depths_from_snapshot(c, host_out);
  return AMOE_OK;
}

amoe_status amoe_box_depths(amoe_ctx_t c, uint32_t* host_out, void* stream) {
  if (!c || !host_out) return AMOE_EINVAL;
  for (int r = 0; r < c->cfg.G; ++r)
    if (!c->dc.peer[r]) return AMOE_EPEER;
  cudaStream_t s = (cudaStream_t)stream;
  c->launches += launch_peer_depths(c->dc, s);
  CK(cudaMemcpyAsync(host_out, c->ws + c->lay.gtot, (size_t)c->cfg.L * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AMOE_OK;
}

amoe_status amoe_pick(amoe_ctx_t c, const uint32_t* Q, int policy, int W, float delta, int* layer, int* queue) {
  if (!c || !Q || !layer || !queue || policy < 0 || policy > 2 || W < 0) return AMOE_EINVAL;
  return pick_queue(Q, c->cfg.L, c->H, c->cfg.E + c->cfg.S, policy, W, (double)delta, layer, queue) ? AMOE_IDLE
                                                                                                   : AMOE_OK;
}

amoe_status amoe_schedule(const uint32_t* Q, int n_blocks, int n_queues, int n_experts, int policy, int W,
                          float delta, int* block, int* queue) {
  if (!Q || !block || !queue || n_blocks < 1 || n_queues < 1 || n_experts < 1 || policy < 0 || policy > 2 || W < 0)
    return AMOE_EINVAL;
  return pick_queue(Q, n_blocks, n_queues, n_experts, policy, W, (double)delta, block, queue) ? AMOE_IDLE : AMOE_OK;
}

amoe_status amoe_schedule_global(const uint32_t* Q, const uint32_t* tot, int n_blocks, int n_queues, int n_experts,
                                 int W, float delta, int* block, int* queue) {
  if (!Q || !tot || !block || !queue || n_blocks < 1 || n_queues < 1 || n_experts < 1 || W < 0) return AMOE_EINVAL;
  return pick_queue(Q, n_blocks, n_queues, n_experts, 0, W, (double)delta, block, queue, tot) ? AMOE_IDLE : AMOE_OK;
}

static amoe_status make_group(amoe_ctx* c, const amoe_group* g, int max_tokens, GroupDev* gd, int* wslot) {
  if (!g || g->nq < 1 || g->nq > AMOE_MAX_GROUP || g->rows_cap < kRowAlign || !g->tile || !g->meta || !g->qinfo)
    return AMOE_EINVAL;
  memset(gd, 0, sizeof(*gd));
  gd->nq = g->nq;
  gd->rows_cap = g->rows_cap;
  gd->max_tokens = max_tokens > 0 ? max_tokens : 0;
  if (c->cfg.max_batch > 0 && (gd->max_tokens == 0 || gd->max_tokens > c->cfg.max_batch)) gd->max_tokens = c->cfg.max_batch;
  if (c->exact_caps) {   // amoe_run's pipelined loop: the drain count is the scheduler's
    gd->exact = 1;
    for (int q = 0; q < g->nq; ++q) gd->cap[q] = c->exact_caps[q];
  }
  gd->qinfo = g->qinfo;
  gd->meta = g->meta;
  gd->tile = g->tile;
  gd->out = g->out;
  for (int q = 0; q < g->nq; ++q) {
    const int slot = local_slot(c, g->layer[q], g->expert[q]);
    if (slot < 0) return AMOE_ENOTHOSTED;
    for (int p = 0; p < q; ++p)
      if (gd->qid[p] == slot) return AMOE_EINVAL;   // a queue may appear once per group
    gd->qid[q] = slot;
    if (wslot) wslot[q] = slot * 3;
  }
  return AMOE_OK;
}

amoe_status amoe_rebatch(amoe_ctx_t c, const amoe_group* g, int max_tokens, void* stream) {
  if (!c) return AMOE_EINVAL;
  GroupDev gd;
  amoe_status st = make_group(c, g, max_tokens, &gd, nullptr);
  if (st != AMOE_OK) return st;
  for (int r = 0; r < c->cfg.G; ++r)
    if (!c->dc.peer[r]) return AMOE_EPEER;
  cudaStream_t s = (cudaStream_t)stream;
  StageTimer tm(c, ST_REBATCH, s);
  c->launches += launch_drain(c->dc, gd, s);
  c->launches += launch_gather(c->dc, gd, c->num_sms, s);
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

// a5 + a6 (+ a7 when fuse: the down-GEMM epilogue stores rows straight into the home pools;
// + the a4 gather when gathered: A rows are TMA-gathered from x by token slot, legs read from
// the rings — single GPU, bf16)
static amoe_status expert_ffn(amoe_ctx* c, const amoe_group* g, int fuse, cudaStream_t s, int gathered = 0) {
  GroupDev gd;
  int wslot[AMOE_MAX_GROUP];
  amoe_status st = make_group(c, g, 0, &gd, wslot);
  if (st != AMOE_OK) return st;
  if (!g->act || !g->out) return AMOE_EINVAL;
  for (int q = 0; q < g->nq; ++q)
    if (!c->hosted_flags[wslot[q] / 3]) return AMOE_EINVAL;   // weights not registered
  for (int r = 0; r < c->cfg.G; ++r)
    if (fuse && !c->dc.peer[r]) return AMOE_EPEER;
  if (c->cfg.dtype == AMOE_BF16) {
    // copies: cached_map returns pointers into a vector that later lookups may reallocate
    CUtensorMap mt, ma, mt32, ma32;
    const CUtensorMap* p;
    if (!(p = gathered ? cached_map(c, c->ws + c->lay.x, c->cfg.T_slots, c->cfg.d, 1)
                       : cached_map(c, g->tile, g->rows_cap, c->cfg.d, 128))) return AMOE_ECUDA;
    mt = *p;
    if (!(p = cached_map(c, g->act, g->rows_cap, c->cfg.ff, 128))) return AMOE_ECUDA;
    ma = *p;
    if (!(p = gathered ? cached_map(c, c->ws + c->lay.x, c->cfg.T_slots, c->cfg.d, 1)
                       : cached_map(c, g->tile, g->rows_cap, c->cfg.d, 32))) return AMOE_ECUDA;
    mt32 = *p;
    if (!(p = cached_map(c, g->act, g->rows_cap, c->cfg.ff, 32))) return AMOE_ECUDA;
    ma32 = *p;
    FfnLaunch f;
    f.nq = g->nq;
    f.qinfo = g->qinfo;
    f.wmaps = reinterpret_cast<const CUtensorMap*>(c->ws + c->lay.wmaps);
    for (int q = 0; q < g->nq; ++q) f.wslot[q] = wslot[q];
    f.rows_hint = gathered ? 0 : g->max_rows_hint;
    if (c->exact_caps) {
      f.exact_max_n = 0;
      for (int q = 0; q < g->nq; ++q) f.exact_max_n = std::max(f.exact_max_n, (int)c->exact_caps[q]);
    }
    {
      StageTimer tm(c, ST_GATEUP, s);
      c->launches += launch_ffn_tc(c->dc, f, mt, ma, mt32, ma32, g->act, g->out, g->meta, 0, gathered, c->num_sms, s, 1);
    }
    {
      StageTimer tm(c, ST_DOWN, s);
      c->launches +=
          launch_ffn_tc(c->dc, f, mt, ma, mt32, ma32, g->act, g->out, g->meta, fuse, gathered, c->num_sms, s, 2);
    }
  } else {
    {
      StageTimer tm(c, ST_GATEUP, s);
      c->launches += launch_ffn_simt(c->dc, g->nq, g->qinfo, wslot,
                                     reinterpret_cast<const uint64_t*>(c->ws + c->lay.wptrs), g->tile, g->act, g->out,
                                     c->num_sms, s);
    }
    if (fuse) {   // the exact fp32 mode keeps the separate forward kernel
      StageTimer tm(c, ST_FORWARD, s);
      c->launches += launch_forward(c->dc, gd, c->num_sms, s);
    }
  }
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

amoe_status amoe_expert_ffn(amoe_ctx_t c, const amoe_group* g, void* stream) {
  if (!c) return AMOE_EINVAL;
  return expert_ffn(c, g, 0, (cudaStream_t)stream);
}

amoe_status amoe_expert_ffn_forward(amoe_ctx_t c, const amoe_group* g, void* stream) {
  if (!c) return AMOE_EINVAL;
  return expert_ffn(c, g, 1, (cudaStream_t)stream);
}

// The fused cold path (k_ffn_cold.cu) vs the four-kernel path for a pick whose queues hold at
// most n_max legs each (nq queues): AMOE_COLD=1 forces the fused kernel (n_max <= 128), 0 the
// four-kernel path; by default the fused kernel takes the picks where it measured faster
// (profiles/r02/cold_sweep_v3.log, device time per pick on one B200):
//  * n_max <= 16: every shape (weight streaming dominates; one launch, no grid-wide hand-off);
//  * n_max <= 32: Mixtral-sized experts (d >= 4096) or groups of >= 4 experts.
// d % 256 == 0 (the fused kernel's down tiles are 256 rows).
static bool cold_pick_ok(const amoe_ctx* c, int n_max, int nq) {
  if (c->cfg.dtype != AMOE_BF16 || n_max < 1 || n_max > 128 || c->cfg.d % 256) return false;
  const char* e = getenv("AMOE_COLD");
  if (e && e[0] == '1') return true;
  if (e && e[0] == '0') return false;
  if (n_max <= 16) return true;
  if (n_max <= 32) return c->cfg.d >= 4096 || nq >= 4;
  return false;
}

// a4 + a5 + a6 + a7 in ONE launch for a cold pick (k_ffn_cold.cu): queue q
// drains exactly n[q] (<= 128) legs from ring position start[q] (its consumer head, which the
// scheduler's snapshot gives), gathers, runs the SwiGLU expert, stores into the home pools.
// bf16 only; the group's act buffer holds nq * n_pad rows.
static amoe_status cold_ffn_forward(amoe_ctx* c, const amoe_group* g, const int* n, const uint32_t* start,
                                    cudaStream_t s) {
  GroupDev gd;
  int wslot[AMOE_MAX_GROUP];
  amoe_status st = make_group(c, g, 0, &gd, wslot);
  if (st != AMOE_OK) return st;
  if (c->cfg.dtype != AMOE_BF16 || !g->act || !n || !start || c->cfg.d % 256) return AMOE_EINVAL;
  int nmax = 1;
  for (int q = 0; q < g->nq; ++q) {
    if (n[q] < 0 || n[q] > 128) return AMOE_EINVAL;
    nmax = std::max(nmax, n[q]);
    if (!c->hosted_flags[wslot[q] / 3]) return AMOE_EINVAL;
  }
  const int n_pad = (nmax + 15) / 16 * 16;
  if ((int64_t)g->nq * n_pad > g->rows_cap) return AMOE_EINVAL;
  for (int r = 0; r < c->cfg.G; ++r)
    if (!c->dc.peer[r]) return AMOE_EPEER;
  int ka = 1, kb = 2;
  cold_blocks(c->cfg.d, c->cfg.ff, n_pad, &ka, &kb);
  const CUtensorMap* p;
  if (!(p = cached_map(c, g->act, g->rows_cap, c->cfg.ff, n_pad, kb))) return AMOE_ECUDA;
  const CUtensorMap ma = *p;
  int qid[AMOE_MAX_GROUP];
  for (int q = 0; q < g->nq; ++q) qid[q] = wslot[q] / 3;
  int k;
  {
    StageTimer tm(c, ST_COLD, s);
    k = launch_ffn_cold(c->dc, g->nq, qid, n, start, n_pad, ka, kb, ma, g->act, g->qinfo,
                        reinterpret_cast<const CUtensorMap*>(c->ws + c->lay.wmaps),
                        reinterpret_cast<const CUtensorMap*>(c->ws + c->lay.cmaps), c->num_sms, s);
  }
  if (k < 0) return AMOE_EINVAL;
  c->launches += k;
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

amoe_status amoe_execute_cold(amoe_ctx_t c, const amoe_group* g, const uint32_t* start, const int32_t* n,
                              void* stream) {
  if (!c || !g || g->nq < 1 || g->nq > AMOE_MAX_GROUP) return AMOE_EINVAL;
  return cold_ffn_forward(c, g, n, start, (cudaStream_t)stream);
}

amoe_status amoe_rebatch_ffn_forward(amoe_ctx_t c, const amoe_group* g, int max_tokens, void* stream) {
  if (!c) return AMOE_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (g && g->nq >= 1 && g->nq <= AMOE_MAX_GROUP && cold_pick_ok(c, g->max_rows_hint, g->nq)) {
    // cold pick: every queue drains its published depth, at most the hint (and max_tokens /
    // cfg.max_batch); the heads and depths come from a counter snapshot (synchronises s)
    int cap = g->max_rows_hint;
    if (max_tokens > 0) cap = std::min(cap, max_tokens);
    if (c->cfg.max_batch > 0) cap = std::min(cap, c->cfg.max_batch);
    GroupDev gd;
    int wslot[AMOE_MAX_GROUP];
    amoe_status st = make_group(c, g, 0, &gd, wslot);
    if (st != AMOE_OK) return st;
    if ((st = snapshot(c, s)) != AMOE_OK) return st;
    const uint32_t* qs = c->pinned + c->lay.qctr / 4;
    int n[AMOE_MAX_GROUP];
    uint32_t start[AMOE_MAX_GROUP];
    for (int q = 0; q < g->nq; ++q) {
      const uint32_t* e = qs + 4 * (wslot[q] / 3);
      n[q] = (int)std::min<uint32_t>(e[1] - e[2], (uint32_t)cap);
      start[q] = e[2];
    }
    return cold_ffn_forward(c, g, n, start, s);
  }
  // The TMA tile::gather4 variant of the fused gather (AMOE_FUSED_GATHER=1) is correct (tests)
  // but slow on B200: each A row is re-read by every N tile of its raster group and gather4
  // moves ~6.6 B/cycle/SM vs >40 for tiled loads (profiles/r01_fused_gather.md).
  // AMOE_CP_GATHER=1 (one GPU, bf16, CTA-pair kernel, hot picks): the gate/up producer warp
  // copies the legs' x rows into its A stages with cp.async (16-B chunks, L2 hits after the first
  // N tile) instead of a gather kernel materialising the tile (2·d·2 HBM bytes per leg); the GEMMs
  // read the drained legs from the rings. Correct (bitwise equal to the materialised path) but
  // slower on B200: the LSU gather holds the gate/up GEMM at ~0.68 of the tensor pipe against
  // 0.97-0.98 with tiled TMA A loads (Mixtral 1.49 vs 1.84 M token-layers/s, DeepSeek 6.4 vs
  // 7.3 M), so the materialised gather stays the default. Peer rows (G > 1)
  // never take it: an A row is re-read by every N tile of its raster group.
  const char* fg = getenv("AMOE_FUSED_GATHER");
  const char* cg = getenv("AMOE_CP_GATHER");
  const char* e1 = getenv("AMOE_FFN_1CTA");
  const bool cp_gather = (cg && cg[0] == '1') && !(fg && fg[0] == '1') && c->cfg.G == 1 &&
                         c->cfg.dtype == AMOE_BF16 && c->cfg.d % 256 == 0 && c->num_sms >= 2 &&
                         !(e1 && e1[0] == '1') && g && (g->max_rows_hint == 0 || g->max_rows_hint > 128) &&
                         (uint64_t)c->cfg.T_slots * (uint64_t)c->cfg.d * 2u < (1ull << 32);
  if (cp_gather || (fg && fg[0] == '1' && c->cfg.G == 1 && c->cfg.dtype == AMOE_BF16)) {
    // a4 drain only; the gather happens inside the gate/up GEMM's A-operand load
    GroupDev gd;
    amoe_status st = make_group(c, g, max_tokens, &gd, nullptr);
    if (st != AMOE_OK) return st;
    {
      StageTimer tm(c, ST_REBATCH, s);
      c->launches += launch_drain(c->dc, gd, s);
    }
    return expert_ffn(c, g, 1, s, cp_gather ? 2 : 1);
  }
  amoe_status st = amoe_rebatch(c, g, max_tokens, s);
  if (st != AMOE_OK) return st;
  return expert_ffn(c, g, 1, s, 0);
}

amoe_status amoe_forward(amoe_ctx_t c, const amoe_group* g, void* stream) {
  if (!c) return AMOE_EINVAL;
  GroupDev gd;
  amoe_status st = make_group(c, g, 0, &gd, nullptr);
  if (st != AMOE_OK) return st;
  if (!g->out) return AMOE_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  StageTimer tm(c, ST_FORWARD, s);
  c->launches += launch_forward(c->dc, gd, c->num_sms, s);
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

amoe_status amoe_combine(amoe_ctx_t c, int retire_pass, void* stream) {
  if (!c) return AMOE_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  DevCtx dc = c->dc;
  if (!dc.router) { dc.n_tab = 1; }
  StageTimer tm(c, ST_COMBINE, s);
  c->launches += launch_combine(dc, retire_pass, c->num_sms, s);
  c->last_stream = s;
  CK(cudaGetLastError());
  return AMOE_OK;
}

amoe_status amoe_scratch_group(amoe_ctx_t c, amoe_group* g) {
  if (!c || !g) return AMOE_EINVAL;
  memset(g, 0, sizeof(*g));
  g->rows_cap = c->lay.rows_cap;
  g->tile = c->ws + c->lay.s_tile;
  g->meta = reinterpret_cast<amoe_leg*>(c->ws + c->lay.s_meta);
  g->qinfo = reinterpret_cast<int32_t*>(c->ws + c->lay.s_qinfo);
  g->act = c->ws + c->lay.s_act;
  g->out = c->ws + c->lay.s_out;
  return AMOE_OK;
}

amoe_status amoe_check(amoe_ctx_t c) {
  if (!c) return AMOE_EINVAL;
  CK(cudaDeviceSynchronize());
  uint32_t e = 0;
  CK(cudaMemcpy(&e, c->ws + c->lay.err, 4, cudaMemcpyDeviceToHost));
  return e ? AMOE_EDEVICE : AMOE_OK;
}

amoe_status amoe_error_info(amoe_ctx_t c, uint32_t info[4]) {
  if (!c || !info) return AMOE_EINVAL;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(info, c->ws + c->lay.err, 16, cudaMemcpyDeviceToHost));
  return AMOE_OK;
}

amoe_status amoe_clear_error(amoe_ctx_t c) {
  if (!c) return AMOE_EINVAL;
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(c->ws + c->lay.err, 0, 16));
  // abort marks peers stored into this rank's done[] slots (multi-GPU fault propagation)
  CK(cudaMemset(c->ws + c->lay.done, 0, 64));
  return AMOE_OK;
}

amoe_status amoe_get_buffer(amoe_ctx_t c, int which, void** ptr, size_t* bytes) {
  if (!c || !ptr || !bytes) return AMOE_EINVAL;
  const uint64_t T = c->cfg.T_slots, d = c->cfg.d, es = c->dc.esize, KS = c->dc.KS, K = c->cfg.K;
  uint64_t off, n;
  switch (which) {
    case AMOE_BUF_H: off = c->lay.h; n = T * d * es; break;
    case AMOE_BUF_X: off = c->lay.x; n = T * d * es; break;
    case AMOE_BUF_POOL: off = c->lay.pool; n = T * KS * d * es; break;
    case AMOE_BUF_TOK_W: off = c->lay.tok_w; n = T * K * 4; break;
    case AMOE_BUF_TOK_IDX: off = c->lay.tok_idx; n = T * K * 4; break;
    case AMOE_BUF_TOK_LAYER: off = c->lay.tok_layer; n = T * 4; break;
    case AMOE_BUF_TOK_PASS: off = c->lay.tok_pass; n = T * 4; break;
    case AMOE_BUF_RINGS: off = c->lay.rings; n = (uint64_t)c->cfg.L * c->H * c->dc.ring_cap * 16; break;
    case AMOE_BUF_QCTR: off = c->lay.qctr; n = (uint64_t)c->cfg.L * c->H * 16; break;
    case AMOE_BUF_STATS: off = c->lay.stats; n = 64; break;
    case AMOE_BUF_SCRATCH: off = c->lay.s_tile; n = c->lay.total - c->lay.s_tile; break;
    case AMOE_BUF_TOK_TIME: off = c->lay.tok_time; n = T * 16; break;
    default: return AMOE_EINVAL;
  }
  *ptr = c->ws + off;
  *bytes = n;
  return AMOE_OK;
}

// Latch a host-detected fault into the device error word (first fault wins, as on the device).
static void host_latch(amoe_ctx* c, uint32_t code, uint32_t a0, uint32_t a1, uint32_t a2, cudaStream_t s) {
  uint32_t cur = 0;
  cudaStreamSynchronize(s);
  cudaMemcpy(&cur, c->ws + c->lay.err, 4, cudaMemcpyDeviceToHost);
  if (cur) return;
  const uint32_t v[4] = {code, a0, a1, a2};
  cudaMemcpy(c->ws + c->lay.err, v, 16, cudaMemcpyHostToDevice);
}

// published depth (snapshot) of the group's j-th queue
static int32_t group_rows(const amoe_ctx* c, const amoe_group& g, int j, const uint32_t* Q, int H) {
  const int lq = g.expert[j] >= c->cfg.E ? c->Hr + (g.expert[j] - c->cfg.E) : c->dc.lq[g.expert[j]];
  return (int32_t)Q[(size_t)g.layer[j] * H + lq];
}

// local queue index (l*H + lq) of the group's j-th queue
static int group_qidx(const amoe_ctx* c, const amoe_group& g, int j, int H) {
  const int lq = g.expert[j] >= c->cfg.E ? c->Hr + (g.expert[j] - c->cfg.E) : c->dc.lq[g.expert[j]];
  return g.layer[j] * H + lq;
}

constexpr int kSmallQueue = 16;   // legs: a queue this small is pure weight streaming (§5.4)

// consumer head (snapshot) of the group's j-th queue
static uint32_t group_head(const amoe_ctx* c, const amoe_group& g, int j, int H) {
  const int lq = g.expert[j] >= c->cfg.E ? c->Hr + (g.expert[j] - c->cfg.E) : c->dc.lq[g.expert[j]];
  return c->pinned[c->lay.qctr / 4 + 4 * ((size_t)g.layer[j] * H + lq) + 2];
}

amoe_status amoe_run(amoe_ctx_t c, const amoe_run_params* p, int retire_pass, amoe_run_stats* stats, void* stream) {
  if (!c || !p || p->policy < 0 || p->policy > AMOE_DEFRAG_GLOBAL || p->W < 0) return AMOE_EINVAL;
  for (int r = 0; r < c->cfg.G; ++r)
    if (!c->dc.peer[r]) return AMOE_EPEER;
  if (!c->dc.router && !c->dc.gate_on) return AMOE_EINVAL;
  if (c->direct && c->cfg.G > 1) {
    // direct forwarding at G > 1 routes with the router gate: every layer needs one here
    for (int l = 0; l < c->cfg.L; ++l)
      if ((int)c->gate_set.size() < c->cfg.L || !c->gate_set[l]) return AMOE_EINVAL;
  }
  for (size_t i = 0; i < c->hosted_flags.size(); ++i)
    if (!c->hosted_flags[i]) {
      // every hosted queue needs weights (routed experts of this rank and the shared experts)
      const int q = (int)(i % c->H);
      if (q < c->Hr) {
        bool exists = false;
        for (int e = 0; e < c->cfg.E; ++e) exists |= (c->dc.owner[e] == c->cfg.rank && c->dc.lq[e] == q);
        if (!exists) continue;
      }
      return AMOE_EINVAL;
    }
  cudaStream_t s = (cudaStream_t)stream;
  c->last_stream = s;
  // the per-pick drain counts (c->exact_caps) point into this frame: cleared on every return,
  // including the error returns between a pick's launches, so a later public amoe_rebatch call
  // never reads a dead pick's caps
  struct ExactCapsReset {
    amoe_ctx* c;
    ~ExactCapsReset() { c->exact_caps = nullptr; }
  } exact_caps_reset{c};
  amoe_run_stats rs{};
  const uint32_t epoch = ++c->epoch;
  const int64_t expected = c->admitted;
  c->admitted = 0;
  amoe_group g;
  amoe_scratch_group(c, &g);
  const int L = c->cfg.L, H = c->H;
  std::vector<uint32_t> Q((size_t)L * H);
  amoe_status st = snapshot(c, s);
  if (st != AMOE_OK) return st;
  log_executions(c, true);
  const uint64_t* s0 = reinterpret_cast<const uint64_t*>(reinterpret_cast<const char*>(c->pinned) + c->lay.stats);
  // merged0: with direct forwarding at G > 1 a peer may already merge this home's tokens before
  // this rank's first snapshot, so the baseline is where the previous run left the counter
  const uint64_t retired0 = s0[1], legs0 = s0[2];
  const uint64_t merged0 = (c->direct && c->cfg.G > 1) ? c->merged_seen : s0[0];
  bool announced = false;
  int idle_streak = 0;
  // AMOE_SYNC: the layer this rank may run, and whether it has arrived at that layer's barrier
  const bool sync = p->policy == AMOE_SYNC;
  // G > 1, asynchronous policies: two opt-in changes to what the scheduler sees when the GPU
  // goes idle (both turn the pipelined loop off):
  // - merge first (AMOE_COMBINE_FIRST=1): pending merges (tokens whose last legs came back from
  //   other ranks) run before the next pick, so their next-layer legs join it;
  // - grow wait (AMOE_GROW_WAIT=<us>): a pick is deferred while its layer's hosted depth still
  //   grows between polls (legs streaming in from a peer's merge), at most that long.
  // Round 1 measured them +3-23 % on the G-rank emulation for ranks hosting >= 2 experts and made
  // them the default there; with round 2's pipelined loop the pipelined Algorithm 1 is ahead
  // (Mixtral G = 2 1.30 vs 1.21 M, G = 4 1.06 vs 1.03 M; box-wide lookahead 1.31 / 1.09 M;
  // profiles/r02/g_emulate_final.log), so both are off by default. Deferrals count as idle.
  const char* cf_env = getenv("AMOE_COMBINE_FIRST");
  const bool combine_first = c->cfg.G > 1 && !sync && p->max_picks == 0 && cf_env && cf_env[0] == '1';
  int64_t grow_ns = 0;
  if (const char* ge = getenv("AMOE_GROW_WAIT")) grow_ns = (int64_t)(atof(ge) * 1e3);
  if (c->cfg.G == 1 || sync || p->max_picks > 0) grow_ns = 0;
  std::vector<uint64_t> prev_depth(grow_ns > 0 ? c->cfg.L : 0, 0);
  int grow_layer = -1;
  auto grow_t0 = std::chrono::steady_clock::now();
  // opt-in (AMOE_MIXED_SPLIT=1): a pick mixing small and hot queues runs the small ones in the
  // fused cold kernel and the rest on the tensor-core path; measured neutral to -4 % on the
  // DeepSeek waves (T = 512: 1.27 -> 1.22 M; larger T never mixes, profiles/r02/mixed_split_ab.md)
  const char* ms_env = getenv("AMOE_MIXED_SPLIT");
  const bool mixed_split = !c->direct && ms_env && ms_env[0] == '1';
  int sync_layer = c->start_layer;
  bool sync_arrived = false;
  // barrier flag value: (run epoch, barrier index + 1), so ranks agree without shared history
  auto bar_tag = [&](int64_t b) { return (epoch << 16) | (uint32_t)((b + 1) & 0xffff); };
  using clk = std::chrono::steady_clock;
  const auto t_run0 = clk::now();
  auto finish = [&](amoe_run_stats* out) {
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);   // no snapshot copy outlives the run
    rs.wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t_run0).count();
    if (out) *out = rs;
  };
  // stepping mode (max_picks > 0, single rank): return after max_picks picks or as soon as
  // nothing is runnable — the caller admits arrivals in between (open-loop serving); no
  // quiescence protocol, no lost-leg verdict
  const bool stepping = p->max_picks > 0;
  // stepping has no layer barrier (the lockstep layer would never advance): AMOE_SYNC is closed-loop only
  if (stepping && (c->cfg.G > 1 || sync)) return AMOE_EINVAL;
  // G > 1: a rank that faults stores kAbortEpoch into every peer's done[] slot, and every rank
  // checks those slots at each poll, so one rank's fault ends every rank's amoe_run with
  // AMOE_EDEVICE instead of leaving the others polling for its done flag. AMOE_RUN_TIMEOUT
  // (seconds, default 600; 0 = off) bounds a run whose legs were lost without a latched fault.
  double timeout_s = 600.0;
  if (const char* te = getenv("AMOE_RUN_TIMEOUT")) timeout_s = atof(te);
  auto abort_run = [&](uint32_t code, uint32_t a0, uint32_t a1, uint32_t a2) -> amoe_status {
    if (code) host_latch(c, code, a0, a1, a2, s);
    if (c->cfg.G > 1) {
      c->launches += launch_announce(c->dc, kAbortEpoch, 0, s);
      cudaStreamSynchronize(s);
    }
    finish(stats);
    return AMOE_EDEVICE;
  };
  // AMOE_DEFRAG_GLOBAL at G > 1: every poll first reads the box-wide per-block depths from all
  // ranks' queue counters (peer_depths_kernel -> gtot, inside the snapshot range)
  const bool global_look = p->policy == AMOE_DEFRAG_GLOBAL && c->cfg.G > 1;
  // Pipelined picks (asynchronous policies, closed loop): the host decides pick k + 1 while pick k
  // runs, instead of waiting for the stream after every pick. Queue depths come from the newest
  // counter snapshot that has landed (copied asynchronously behind each pick) minus what the
  // host itself has drained since — every drain takes exactly the count the host decided
  // (GroupDev::exact / the cold kernel's n), so the host's consumer heads are exact and its depth
  // estimate never exceeds the published count. At most two picks are in flight; stale views only
  // delay decisions (idleness and quiescence are judged on a fresh view). AMOE_PIPELINE=0 off.
  const char* pl_env = getenv("AMOE_PIPELINE");
  const bool pipe = !sync && !stepping && grow_ns == 0 && !combine_first &&
                    !(pl_env && pl_env[0] == '0');
  const int NQ = L * H;
  std::vector<uint32_t> head_host, commit_seen;
  struct Outst { int buf; };
  std::vector<Outst> outst;        // FIFO of snapshots in flight (oldest first)
  int view_buf = -1;               // snapshot buffer the loop reads (pipelined)
  bool dirty = false, want_fresh = false;
  uint64_t launches_at_view = 0;   // c->launches when the current view's copy was issued
  uint64_t combine_launch_mark = 0;  // c->launches right after the last combine was issued
  if (pipe) {
    for (int i = 0; i < 3; ++i)
      if (!c->snapbuf[i] && cudaMallocHost(&c->snapbuf[i], c->snap_bytes) != cudaSuccess) return AMOE_ECUDA;
    for (int i = 0; i < 6; ++i)
      if (!c->snapev[i] && cudaEventCreateWithFlags(&c->snapev[i], cudaEventDisableTiming) != cudaSuccess)
        return AMOE_ECUDA;
    if (!c->copy_stream && cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      return AMOE_ECUDA;
    memcpy(c->snapbuf[0], c->pinned, c->snap_bytes);
    view_buf = 0;
    const uint32_t* qs = c->pinned + c->lay.qctr / 4;
    head_host.resize(NQ);
    commit_seen.resize(NQ);
    for (int i = 0; i < NQ; ++i) { head_host[i] = qs[4 * i + 2]; commit_seen[i] = qs[4 * i + 1]; }
    launches_at_view = c->launches;
  }
  auto issue_snapshot = [&]() -> amoe_status {
    // a free buffer: not the view, not in flight
    int b = 0;
    for (; b < 3; ++b) {
      bool busy = b == view_buf;
      for (const auto& o : outst) busy |= o.buf == b;
      if (!busy) break;
    }
    if (global_look) c->launches += launch_peer_depths(c->dc, s);
    // the copy runs on a side stream behind an event: the compute stream goes straight from this
    // pick's merge to the next pick's kernels, so programmatic dependent launch overlaps their
    // prologues (a copy between them on the same stream would serialise every boundary). The
    // copy may also see later picks' counter updates: every field the loop reads is monotone or
    // re-checked (published counts, merge / retire counts, flags)
    CK(cudaEventRecord(c->snapev[3 + b], s));
    CK(cudaStreamWaitEvent(c->copy_stream, c->snapev[3 + b], 0));
    CK(cudaMemcpyAsync(c->snapbuf[b], c->ws, c->snap_bytes, cudaMemcpyDeviceToHost, c->copy_stream));
    CK(cudaEventRecord(c->snapev[b], c->copy_stream));
    outst.push_back({b});
    return AMOE_OK;
  };
  std::vector<uint64_t> outst_launches;   // c->launches when each in-flight copy was issued
  uint64_t issued_mark = c->launches;     // c->launches when the newest copy was issued
  auto consume = [&](bool all) -> amoe_status {
    while (!outst.empty()) {
      const int b = outst.front().buf;
      if (all || outst.size() >= 2) {
        CK(cudaEventSynchronize(c->snapev[b]));
      } else {
        const cudaError_t q = cudaEventQuery(c->snapev[b]);
        if (q == cudaErrorNotReady) break;
        if (q != cudaSuccess) return AMOE_ECUDA;
      }
      view_buf = b;
      launches_at_view = outst_launches.front();
      outst.erase(outst.begin());
      outst_launches.erase(outst_launches.begin());
      const uint32_t* qs = c->snapbuf[b] + c->lay.qctr / 4;
      for (int i = 0; i < NQ; ++i)
        if ((int32_t)(qs[4 * i + 1] - commit_seen[i]) > 0) commit_seen[i] = qs[4 * i + 1];
    }
    return AMOE_OK;
  };
  for (;;) {
    if (pipe) {
      dirty = dirty || (uint64_t)c->launches != issued_mark;
      if (dirty) {
        if ((st = issue_snapshot()) != AMOE_OK) return st;
        issued_mark = c->launches;
        outst_launches.push_back(c->launches);
        dirty = false;
      }
      if ((st = consume(want_fresh)) != AMOE_OK) return st;
      want_fresh = false;
    } else {
      if (global_look) c->launches += launch_peer_depths(c->dc, s);
      st = snapshot(c, s);   // waits for this rank's previous launches: the GPU is idle from here
      if (st != AMOE_OK) return st;
    }
    // fresh: the view reflects every launch this rank issued
    const bool fresh = !pipe || (outst.empty() && !dirty && launches_at_view == (uint64_t)c->launches);
    const auto t_poll = clk::now();
    const char* snap = pipe ? reinterpret_cast<const char*>(c->snapbuf[view_buf]) : reinterpret_cast<const char*>(c->pinned);
    if (*reinterpret_cast<const uint32_t*>(snap + c->lay.err)) return abort_run(0, 0, 0, 0);
    if (c->cfg.G > 1) {
      const uint32_t* dn = reinterpret_cast<const uint32_t*>(snap + c->lay.done);
      for (int r = 0; r < c->cfg.G; ++r)
        if (r != c->cfg.rank && dn[r] == kAbortEpoch) return abort_run(F_PEER_ABORT, (uint32_t)r, 0, 0);
      const double el = std::chrono::duration<double>(t_poll - t_run0).count();
      if (timeout_s > 0 && el > timeout_s) {
        const uint64_t* sv0 = reinterpret_cast<const uint64_t*>(snap + c->lay.stats);
        return abort_run(F_RUN_TIMEOUT, (uint32_t)el, (uint32_t)(sv0[0] - merged0), (uint32_t)expected);
      }
    }
    const uint64_t* sv = reinterpret_cast<const uint64_t*>(snap + c->lay.stats);
    if (!pipe) log_executions(c, false);   // pipelined: executions are logged as they are issued
    if (sync && !announced && !stepping) {
      const uint32_t* flags = reinterpret_cast<const uint32_t*>(snap + c->lay.done) + AMOE_MAX_G;
      if (!sync_arrived && (int64_t)(sv[0] - merged0) >= expected * (int64_t)(rs.barriers + 1) &&
          (int64_t)(sv[1] - retired0) < expected) {   // the last layer of the run has no barrier
        // every homed token merged layer sync_layer: arrive at the barrier (flag in every peer)
        c->launches += launch_announce(c->dc, bar_tag(rs.barriers), AMOE_MAX_G, s);
        rs.kernel_launches += 1;
        sync_arrived = true;
        continue;
      }
      if (sync_arrived) {
        // a rank whose tokens all retired (done == epoch) has nothing left to merge at this layer
        const uint32_t* done = reinterpret_cast<const uint32_t*>(snap + c->lay.done);
        bool all = true;
        for (int r = 0; r < c->cfg.G; ++r)
          all &= (int32_t)(flags[r] - bar_tag(rs.barriers)) >= 0 || done[r] == epoch;
        if (all) {   // no leg of sync_layer is left anywhere: take the next layer
          rs.barriers += 1;
          sync_layer = (sync_layer + 1) % L;
          sync_arrived = false;
          continue;
        }
      }
    }
    if (!stepping && !announced && (int64_t)(sv[1] - retired0) >= expected) {
      c->launches += launch_announce(c->dc, epoch, 0, s);
      rs.kernel_launches += 1;
      announced = true;
      continue;
    }
    if (announced) {
      const uint32_t* done = reinterpret_cast<const uint32_t*>(snap + c->lay.done);
      bool all = true;
      for (int r = 0; r < c->cfg.G; ++r) all &= done[r] == epoch;
      if (all) {
        c->merged_seen = sv[0];
        rs.token_layers = (int64_t)(sv[0] - merged0);
        rs.legs = (int64_t)(sv[2] - legs0);
        break;
      }
    }
    if (pipe)
      for (int i = 0; i < NQ; ++i) Q[i] = commit_seen[i] - head_host[i];
    else
      depths_from_snapshot(c, Q.data());
    if (sync)   // lockstep: only the current layer's queues are eligible
      for (int bb = 0; bb < L; ++bb)
        if (bb != sync_layer) std::fill(Q.begin() + (size_t)bb * H, Q.begin() + (size_t)(bb + 1) * H, 0u);
    const uint32_t* cc = reinterpret_cast<const uint32_t*>(snap + c->lay.cctr);
    // pending merges; a view taken before the last combine launch no longer tells
    const uint32_t cpend = (pipe && combine_launch_mark > launches_at_view) ? 0u : cc[1] - cc[2];
    if (combine_first && cpend > 0) {
      // merge the tokens whose last legs arrived from other ranks before picking: their next
      // layer's legs join the queues first, so the pick drains one batch instead of a fragment
      const int64_t l0 = c->launches;
      if ((st = amoe_combine(c, retire_pass, s)) != AMOE_OK) return st;
      rs.kernel_launches += c->launches - l0;
      idle_streak = 0;
      continue;
    }
    int b = -1, q = -1;
    const int pol = sync ? AMOE_MTFS : p->policy == AMOE_DEFRAG_GLOBAL ? AMOE_DEFRAG : p->policy;
    const uint32_t* look = global_look ? reinterpret_cast<const uint32_t*>(snap + c->lay.gtot) : nullptr;
    bool work = pick_queue(Q.data(), L, H, c->cfg.E + c->cfg.S, pol, p->W, (double)p->delta, &b, &q, look) == 0;
    if (work && grow_ns > 0) {
      uint64_t depth = 0;
      for (int j = 0; j < H; ++j) depth += Q[(size_t)b * H + j];
      const bool grew = depth > prev_depth[b];
      for (int l = 0; l < L; ++l) {
        uint64_t t = 0;
        for (int j = 0; j < H; ++j) t += Q[(size_t)l * H + j];
        prev_depth[l] = t;
      }
      const auto now = clk::now();
      if (grow_layer != b) { grow_layer = b; grow_t0 = now; }
      if (grew && std::chrono::duration_cast<std::chrono::nanoseconds>(now - grow_t0).count() < grow_ns) {
        std::this_thread::sleep_for(std::chrono::microseconds(5));
        rs.idle_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t_poll).count();
        continue;
      }
      grow_layer = -1;
    }
    if (work) {
      g.nq = 0;
      if (p->grouped) {
        for (int j = 0; j < H && g.nq < AMOE_MAX_GROUP; ++j)
          if (Q[(size_t)b * H + j] > 0) {
            g.layer[g.nq] = b;
            g.expert[g.nq] = j < c->Hr ? -1 : c->cfg.E + (j - c->Hr);
            if (j < c->Hr)
              for (int e = 0; e < c->cfg.E; ++e)
                if (c->dc.owner[e] == c->cfg.rank && c->dc.lq[e] == j) g.expert[g.nq] = e;
            ++g.nq;
          }
      } else {
        g.layer[0] = b;
        g.expert[0] = q < c->Hr ? -1 : c->cfg.E + (q - c->Hr);
        if (q < c->Hr)
          for (int e = 0; e < c->cfg.E; ++e)
            if (c->dc.owner[e] == c->cfg.rank && c->dc.lq[e] == q) g.expert[0] = e;
        g.nq = 1;
      }
      // performance hint for the FFN kernel choice: the largest published queue at this pick
      // (a drain takes at least that many; single-rank waves take exactly that many)
      g.max_rows_hint = 0;
      for (int j = 0; j < g.nq; ++j) g.max_rows_hint = std::max(g.max_rows_hint, group_rows(c, g, j, Q.data(), H));
      const int64_t l0 = c->launches;
      // cold pick: every queue drains <= 128 legs (its snapshot depth, or the max_batch cap),
      // from its consumer head in the snapshot
      int cold_caps[AMOE_MAX_GROUP];
      uint32_t cold_start[AMOE_MAX_GROUP];
      int cold_max = 0;
      for (int j = 0; j < g.nq; ++j) {
        int cap = group_rows(c, g, j, Q.data(), H);
        if (c->cfg.max_batch > 0) cap = std::min(cap, c->cfg.max_batch);
        cold_caps[j] = cap;
        cold_start[j] = pipe ? head_host[group_qidx(c, g, j, H)] : group_head(c, g, j, H);
        cold_max = std::max(cold_max, cap);
      }
      const bool cold_pick = cold_pick_ok(c, cold_max, g.nq);
      int n_small = 0;
      for (int j = 0; j < g.nq; ++j) n_small += cold_caps[j] <= kSmallQueue;
      // pipelined: every drain of this pick takes exactly the host's count (cold_caps)
      if (pipe) c->exact_caps = cold_caps;
      if (c->direct) {
        // top-1 direct forwarding (f3): drain + gather, SwiGLU expert into the group's out rows,
        // then this rank merges, normalises, routes and scatters each token itself
        if ((st = amoe_rebatch(c, &g, 0, s)) != AMOE_OK) return st;
        if ((st = expert_ffn(c, &g, 0, s)) != AMOE_OK) return st;
        GroupDev gd;
        if ((st = make_group(c, &g, 0, &gd, nullptr)) != AMOE_OK) return st;
        {
          StageTimer tm(c, ST_COMBINE, s);
          c->launches += launch_direct_merge(c->dc, gd, retire_pass, c->num_sms, s);
        }
        CK(cudaGetLastError());
        rs.picks += 1;
      } else if (!cold_pick && mixed_split && c->cfg.dtype == AMOE_BF16 && n_small >= 2 && n_small < g.nq) {
        // a pick mixing small queues (<= 16 legs: pure weight streaming) with hot ones: the small
        // queues run in one fused cold launch, the hot ones on the tensor-core path behind it
        amoe_group gc = g, gh = g;
        gc.nq = gh.nq = 0;
        int cc_caps[AMOE_MAX_GROUP], ch_caps[AMOE_MAX_GROUP];
        uint32_t cc_start[AMOE_MAX_GROUP];
        for (int j = 0; j < g.nq; ++j) {
          const bool small = cold_caps[j] <= kSmallQueue;
          amoe_group& t = small ? gc : gh;
          t.layer[t.nq] = g.layer[j];
          t.expert[t.nq] = g.expert[j];
          if (small) { cc_caps[gc.nq] = cold_caps[j]; cc_start[gc.nq] = cold_start[j]; }
          else ch_caps[gh.nq] = cold_caps[j];
          ++t.nq;
        }
        gh.max_rows_hint = 1 << 30;   // the hot part stays on the tensor-core path
        c->exact_caps = nullptr;
        if ((st = cold_ffn_forward(c, &gc, cc_caps, cc_start, s)) != AMOE_OK) return st;
        if (pipe) c->exact_caps = ch_caps;
        if ((st = amoe_rebatch(c, &gh, 0, s)) != AMOE_OK) return st;
        if ((st = expert_ffn(c, &gh, 1, s)) != AMOE_OK) return st;
        rs.picks += 1;
      } else if (cold_pick) {
        // every queue of the pick is cold: the fused one-launch path, each queue drained up to
        // the depth this pick saw (its published prefix at the snapshot)
        if ((st = cold_ffn_forward(c, &g, cold_caps, cold_start, s)) != AMOE_OK) return st;
        rs.picks += 1;
      } else {
        if ((st = amoe_rebatch_ffn_forward(c, &g, 0, s)) != AMOE_OK) return st;
        rs.picks += 1;
      }
      c->exact_caps = nullptr;
      if (pipe)
        for (int j = 0; j < g.nq; ++j) {
          const int qi = group_qidx(c, g, j, H);
          head_host[qi] += (uint32_t)cold_caps[j];
          if (c->prof && cold_caps[j] > 0) { c->exec_log.push_back(qi); c->exec_log.push_back(cold_caps[j]); }
        }
      if (!c->direct && (st = amoe_combine(c, retire_pass, s)) != AMOE_OK) return st;
      combine_launch_mark = c->launches;
      rs.kernel_launches += c->launches - l0;
      rs.queues_run += g.nq;
      idle_streak = 0;
    } else if (cpend > 0) {
      const int64_t l0 = c->launches;
      if ((st = amoe_combine(c, retire_pass, s)) != AMOE_OK) return st;
      combine_launch_mark = c->launches;
      rs.kernel_launches += c->launches - l0;
      idle_streak = 0;
    } else if (!fresh) {
      // nothing decidable on a stale view: wait for the newest snapshot (the in-flight picks'
      // merges may have queued the next layer) before judging idleness
      want_fresh = true;
    } else {
      rs.idle_polls += 1;
      if (stepping) {
        rs.token_layers = (int64_t)(sv[0] - merged0);
        rs.legs = (int64_t)(sv[2] - legs0);
        break;
      }
      if (c->cfg.G == 1 && !announced && !sync_arrived) {
        // single GPU: nothing queued and tokens not retired means a lost leg. Name the first
        // stranded token (admitted, not retired: SPEC.md L401's audit) in the error word:
        // F_LOST_LEG (slot, layer, columns of its legs that came back)
        rs.token_layers = (int64_t)(sv[0] - merged0);
        const int T = c->cfg.T_slots;
        std::vector<uint64_t> tt((size_t)2 * T);
        std::vector<uint32_t> ld(T);
        std::vector<int32_t> tl(T);
        cudaMemcpy(tt.data(), c->ws + c->lay.tok_time, tt.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(ld.data(), c->ws + c->lay.legs_done, ld.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(tl.data(), c->ws + c->lay.tok_layer, tl.size() * 4, cudaMemcpyDeviceToHost);
        for (int t = 0; t < T; ++t)
          if (tt[2 * t] != 0 && tt[2 * t + 1] == 0) {
            host_latch(c, F_LOST_LEG, (uint32_t)t, (uint32_t)tl[t], ld[t], s);
            break;
          }
        finish(stats);
        return AMOE_EDEVICE;
      }
      if (++idle_streak > 64) std::this_thread::sleep_for(std::chrono::microseconds(5));
      rs.idle_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t_poll).count();
      if (pipe) { dirty = true; want_fresh = true; }   // poll: a new snapshot next time round
    }
    if (stepping && rs.picks >= p->max_picks) {
      rs.token_layers = (int64_t)(sv[0] - merged0);   // merges observed up to this pick's launch
      rs.legs = (int64_t)(sv[2] - legs0);
      break;
    }
  }
  finish(stats);
  return AMOE_OK;
}

amoe_status amoe_pass_host(amoe_ctx_t c, const void* h0_host, const float* router_host, void* h_out_host, int pass,
                           const amoe_run_params* p, amoe_run_stats* stats, void* stream) {
  const bool gate0 = c && !c->gate_set.empty() && c->gate_set[0];
  if (!c || !h0_host || !h_out_host || !p || (!c->dc.router && !gate0)) return AMOE_EINVAL;
  if (router_host && !c->dc.router) return AMOE_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)c->cfg.T_slots * c->cfg.d * c->dc.esize;
  // all slots, identity order: the slot list lives in the scratch meta area head (int32 iota)
  static_assert(sizeof(amoe_leg) == 16, "leg layout");
  int32_t* slots = reinterpret_cast<int32_t*>(c->ws + c->lay.s_meta);
  if ((uint64_t)c->lay.rows_cap * 16 < (uint64_t)c->cfg.T_slots * 4) return AMOE_EINVAL;
  std::vector<int32_t> iota(c->cfg.T_slots);
  for (int i = 0; i < c->cfg.T_slots; ++i) iota[i] = i;
  CK(cudaMemcpyAsync(slots, iota.data(), iota.size() * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(c->ws + c->lay.h, h0_host, bytes, cudaMemcpyHostToDevice, s));
  if (router_host) {
    const size_t tb = (size_t)c->cfg.L * c->cfg.T_slots * c->cfg.E * sizeof(float);
    float* dst = const_cast<float*>(c->dc.router) + (size_t)(pass % c->dc.n_tab) * c->cfg.L * c->cfg.T_slots * c->cfg.E;
    CK(cudaMemcpyAsync(dst, router_host, tb, cudaMemcpyHostToDevice, s));
  }
  amoe_status st = amoe_token_init(c, slots, c->cfg.T_slots, c->ws + c->lay.h, pass, s);
  if (st != AMOE_OK) return st;
  // layer 0 routes with its gate when it has one, else from the router table
  const float* z0 = gate0 ? nullptr
                          : c->dc.router + (uint64_t)(pass % c->dc.n_tab) * c->cfg.L * c->cfg.T_slots * c->cfg.E;
  if ((st = amoe_enqueue(c, 0, slots, c->cfg.T_slots, z0, nullptr, nullptr, s)) != AMOE_OK) return st;
  CK(cudaStreamSynchronize(s));   // the slot list area is reused as scratch by amoe_run
  if ((st = amoe_run(c, p, pass + 1, stats, s)) != AMOE_OK) return st;
  CK(cudaMemcpyAsync(h_out_host, c->ws + c->lay.h, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return AMOE_OK;
}

amoe_status amoe_profile_enable(amoe_ctx_t c, int enable) {
  if (!c) return AMOE_EINVAL;
  CK(cudaDeviceSynchronize());
  for (auto& r : c->recs) { c->ev_pool.push_back(r.a); c->ev_pool.push_back(r.b); }
  c->recs.clear();
  for (int i = 0; i < 8; ++i) { c->prof_ms[i] = 0; c->prof_n[i] = 0; }
  c->prof = enable != 0;
  c->exec_log.clear();
  return AMOE_OK;
}

amoe_status amoe_exec_log(amoe_ctx_t c, int32_t* out, int cap, int* n_out) {
  if (!c || !n_out || cap < 0 || (cap > 0 && !out)) return AMOE_EINVAL;
  const int n = (int)(c->exec_log.size() / 2);
  *n_out = n;
  std::copy(c->exec_log.begin(), c->exec_log.begin() + 2 * (size_t)std::min(n, cap), out);
  return AMOE_OK;
}

amoe_status amoe_profile_read(amoe_ctx_t c, double* ms_out, int64_t* counts_out) {
  if (!c || !ms_out || !counts_out) return AMOE_EINVAL;
  for (auto& r : c->recs) {
    CK(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    c->prof_ms[r.stage] += ms;
    c->prof_n[r.stage] += 1;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->recs.clear();
  for (int i = 0; i < 8; ++i) { ms_out[i] = c->prof_ms[i]; counts_out[i] = c->prof_n[i]; }
  return AMOE_OK;
}

amoe_status amoe_destroy(amoe_ctx_t c) {
  if (!c) return AMOE_EINVAL;
  for (auto& r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->pinned) cudaFreeHost(c->pinned);
  for (int i = 0; i < 3; ++i)
    if (c->snapbuf[i]) cudaFreeHost(c->snapbuf[i]);
  for (int i = 0; i < 6; ++i)
    if (c->snapev[i]) cudaEventDestroy(c->snapev[i]);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  delete c;
  return AMOE_OK;
}

}  // extern "C"
