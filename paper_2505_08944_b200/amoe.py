"""Thin Python binding of libamoe (include/amoe.h): argument marshalling only.

Every step of the hot path runs in libamoe's CUDA kernels. PyTorch provides device memory,
streams and (multi-GPU) process groups / symmetric memory. If the shared library is missing
this module raises at import-time use — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

MAX_G, MAX_E, MAX_GROUP = 8, 256, 128
BF16, FP32 = 0, 1
DEFRAG, MTFS, FLFS, SYNC, DEFRAG_GLOBAL = 0, 1, 2, 3, 4
POLICIES = {"defrag": DEFRAG, "mtfs": MTFS, "flfs": FLFS, "sync": SYNC, "defrag_global": DEFRAG_GLOBAL}
BUF = dict(h=0, x=1, pool=2, tok_w=3, tok_idx=4, tok_layer=5, tok_pass=6, rings=7, qctr=8, stats=9, scratch=10,
           tok_time=11)
STATUS = {0: "OK", 1: "IDLE", 2: "EINVAL", 3: "ENOTHOSTED", 4: "ECUDA", 5: "EDEVICE", 6: "EPEER", 7: "ENOMEM"}
FAULTS = {1: "ring overflow", 2: "leg count > K+S", 3: "expert index out of range", 4: "not hosted",
          5: "combine ring overflow", 6: "token slot out of range", 7: "stale/unpublished ring entry",
          8: "no router table", 9: "aborted by a peer rank's fault", 10: "amoe_run timeout (G > 1)",
          11: "lost leg: stranded token"}

# AMOE_LIB: load another build of the same library (A/B measurements of two builds in one run)
LIB_PATH = os.environ.get("AMOE_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libamoe.so")


class Config(C.Structure):
    _fields_ = [("L", C.c_int32), ("E", C.c_int32), ("K", C.c_int32), ("S", C.c_int32), ("d", C.c_int32),
                ("ff", C.c_int32), ("G", C.c_int32), ("rank", C.c_int32), ("T_slots", C.c_int32),
                ("dtype", C.c_int32), ("max_batch", C.c_int32), ("rows_cap", C.c_int32),
                ("rms_eps", C.c_float), ("owner", C.c_int32 * MAX_E)]


class Leg(C.Structure):
    _fields_ = [("token_slot", C.c_int32), ("k", C.c_int16), ("home", C.c_int16), ("w", C.c_float),
                ("seq", C.c_uint32)]


class Group(C.Structure):
    _fields_ = [("nq", C.c_int32), ("layer", C.c_int32 * MAX_GROUP), ("expert", C.c_int32 * MAX_GROUP),
                ("rows_cap", C.c_int32), ("tile", C.c_void_p), ("meta", C.c_void_p), ("qinfo", C.c_void_p),
                ("act", C.c_void_p), ("out", C.c_void_p), ("max_rows_hint", C.c_int32)]


class RunParams(C.Structure):
    _fields_ = [("policy", C.c_int32), ("W", C.c_int32), ("delta", C.c_float), ("grouped", C.c_int32),
                ("max_picks", C.c_int32)]


class RunStats(C.Structure):
    _fields_ = [("picks", C.c_int64), ("queues_run", C.c_int64), ("legs", C.c_int64),
                ("token_layers", C.c_int64), ("kernel_launches", C.c_int64), ("idle_polls", C.c_int64),
                ("idle_ns", C.c_int64), ("wall_ns", C.c_int64), ("barriers", C.c_int64)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


EXPORTS = {
    "amoe_workspace_bytes": (C.c_size_t, [C.POINTER(Config)]),
    "amoe_create": (C.c_int, [C.POINTER(Config), C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "amoe_import_peers": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int]),
    "amoe_set_expert": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "amoe_set_router": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "amoe_set_exec_log": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "amoe_set_gate": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "amoe_token_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]),
    "amoe_enqueue": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "amoe_queue_depths": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.c_void_p]),
    "amoe_pick": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.c_int, C.c_int, C.c_float,
                            C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "amoe_schedule": (C.c_int, [C.POINTER(C.c_uint32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float,
                                C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "amoe_set_direct": (C.c_int, [C.c_void_p, C.c_int]),
    "amoe_box_depths": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.c_void_p]),
    "amoe_schedule_global": (C.c_int, [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_float, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "amoe_rebatch": (C.c_int, [C.c_void_p, C.POINTER(Group), C.c_int, C.c_void_p]),
    "amoe_expert_ffn": (C.c_int, [C.c_void_p, C.POINTER(Group), C.c_void_p]),
    "amoe_forward": (C.c_int, [C.c_void_p, C.POINTER(Group), C.c_void_p]),
    "amoe_expert_ffn_forward": (C.c_int, [C.c_void_p, C.POINTER(Group), C.c_void_p]),
    "amoe_rebatch_ffn_forward": (C.c_int, [C.c_void_p, C.POINTER(Group), C.c_int, C.c_void_p]),
    "amoe_execute_cold": (C.c_int, [C.c_void_p, C.POINTER(Group), C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                    C.c_void_p]),
    "amoe_combine": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "amoe_run": (C.c_int, [C.c_void_p, C.POINTER(RunParams), C.c_int, C.POINTER(RunStats), C.c_void_p]),
    "amoe_pass_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(RunParams),
                                 C.POINTER(RunStats), C.c_void_p]),
    "amoe_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "amoe_profile_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "amoe_exec_log": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_int)]),
    "amoe_get_buffer": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "amoe_hosted": (C.c_int, [C.c_void_p]),
    "amoe_ring_cap": (C.c_int, [C.c_void_p]),
    "amoe_local_queue": (C.c_int, [C.c_void_p, C.c_int]),
    "amoe_scratch_group": (C.c_int, [C.c_void_p, C.POINTER(Group)]),
    "amoe_launch_count": (C.c_int64, [C.c_void_p]),
    "amoe_die_info": (C.c_int, [C.POINTER(C.c_int32)]),
    "amoe_check": (C.c_int, [C.c_void_p]),
    "amoe_error_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "amoe_clear_error": (C.c_int, [C.c_void_p]),
    "amoe_status_string": (C.c_char_p, [C.c_int]),
    "amoe_destroy": (C.c_int, [C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libamoe.so (build it with `python -m paper_2505_08944_b200.build`). Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"libamoe.so not found at {path}: run `python -m paper_2505_08944_b200.build` "
                               "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _lib = lib
    return _lib


class AmoeError(RuntimeError):
    def __init__(self, status, what, info=None):
        msg = f"{what}: {STATUS.get(status, status)}"
        if info is not None and info[0]:
            msg += f" (device fault {info[0]} '{FAULTS.get(info[0], '?')}' args {list(info[1:])})"
        super().__init__(msg)
        self.status = status
        self.info = info


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_config(L, E, K, S, d, ff, T_slots, G=1, rank=0, dtype="bf16", max_batch=0, rows_cap=0, owner=None,
                rms_eps=1e-6) -> Config:
    cfg = Config()
    cfg.L, cfg.E, cfg.K, cfg.S, cfg.d, cfg.ff = L, E, K, S, d, ff
    cfg.G, cfg.rank, cfg.T_slots = G, rank, T_slots
    cfg.dtype = BF16 if dtype == "bf16" else FP32
    cfg.max_batch, cfg.rows_cap, cfg.rms_eps = max_batch, rows_cap, rms_eps
    own = [e % G for e in range(E)] if owner is None else list(owner)
    for e in range(E):
        cfg.owner[e] = own[e]
    return cfg


def workspace_bytes(cfg: Config) -> int:
    return int(load().amoe_workspace_bytes(C.byref(cfg)))


def die_info():
    """(SMs on die 0, SMs on die 1) from the library's probe; (n, 0) = no die split detected."""
    c = (C.c_int32 * 2)()
    st = load().amoe_die_info(c)
    if st != 0:
        raise AmoeError(st, "amoe_die_info")
    return int(c[0]), int(c[1])


def schedule(Q, n_experts, policy="defrag", W=4, delta=0.5):
    """Host scheduler (Algorithm 1 / MTFS / FLFS) on a [blocks, queues] depth array; None = idle."""
    import numpy as np
    q = np.ascontiguousarray(Q, dtype=np.uint32)
    b, e = C.c_int(), C.c_int()
    st = load().amoe_schedule(q.ctypes.data_as(C.POINTER(C.c_uint32)), q.shape[0], q.shape[1], n_experts,
                              POLICIES[policy], W, delta, C.byref(b), C.byref(e))
    if st not in (0, 1):
        raise AmoeError(st, "amoe_schedule")
    return None if st == 1 else (b.value, e.value)


def schedule_global(Q_local, block_totals, n_experts, W=4, delta=0.5):
    """Algorithm 1 with a box-wide lookahead (AMOE_DEFRAG_GLOBAL): Q_local [blocks, queues] = this
    GPU's depths, block_totals [blocks] = every GPU's queued legs per block; None = idle."""
    import numpy as np
    q = np.ascontiguousarray(Q_local, dtype=np.uint32)
    t = np.ascontiguousarray(block_totals, dtype=np.uint32)
    assert t.shape == (q.shape[0],)
    b, e = C.c_int(), C.c_int()
    st = load().amoe_schedule_global(q.ctypes.data_as(C.POINTER(C.c_uint32)), t.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     q.shape[0], q.shape[1], n_experts, W, delta, C.byref(b), C.byref(e))
    if st not in (0, 1):
        raise AmoeError(st, "amoe_schedule_global")
    return None if st == 1 else (b.value, e.value)


class GroupBuffers:
    """Caller-owned device buffers of one grouped execution (amoe_group)."""

    def __init__(self, ctx: "Context", rows_cap: int):
        dev, tdt = ctx.device, ctx.torch_dtype
        self.rows_cap = rows_cap
        self.tile = torch.zeros(rows_cap, ctx.d, dtype=tdt, device=dev)
        self.meta = torch.zeros(rows_cap, 4, dtype=torch.int32, device=dev)
        self.qinfo = torch.zeros(3 * MAX_GROUP, dtype=torch.int32, device=dev)
        self.act = torch.zeros(rows_cap, ctx.ff, dtype=tdt, device=dev)
        self.out = torch.zeros(rows_cap, ctx.d, dtype=tdt, device=dev)
        self.g = Group()
        self.g.rows_cap = rows_cap
        self.g.tile, self.g.meta, self.g.qinfo = self.tile.data_ptr(), self.meta.data_ptr(), self.qinfo.data_ptr()
        self.g.act, self.g.out = self.act.data_ptr(), self.out.data_ptr()

    def set_queues(self, pairs, max_rows_hint=0):
        self.g.max_rows_hint = max_rows_hint
        self.g.nq = len(pairs)
        for i, (l, e) in enumerate(pairs):
            self.g.layer[i], self.g.expert[i] = l, e
        return self

    def info(self):
        """(n, row_off, start) per queue, on the host."""
        q = self.qinfo.cpu().numpy()
        nq = self.g.nq
        return q[:nq], q[MAX_GROUP:MAX_GROUP + nq], q[2 * MAX_GROUP:2 * MAX_GROUP + nq]


class Context:
    """One libamoe context (one rank). The workspace is a caller-owned torch uint8 tensor."""

    def __init__(self, cfg: Config, workspace: torch.Tensor | None = None, device=None):
        self.lib = load()
        self.cfg = cfg
        self.device = torch.device(device or "cuda")
        nbytes = workspace_bytes(cfg)
        if nbytes == 0:
            raise AmoeError(2, "amoe_workspace_bytes (invalid config)")
        if workspace is None:
            workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        if workspace.dtype != torch.uint8 or not workspace.is_contiguous() or workspace.device.type != "cuda":
            raise AmoeError(2, "workspace must be a contiguous uint8 CUDA tensor")
        base = workspace.data_ptr()
        pad = (-base) % 256
        if workspace.numel() - pad < nbytes:
            # a short buffer would be silently truncated by the slice below; the library's own
            # size check (AMOE_ENOMEM) only sees the byte count passed to amoe_create
            raise AmoeError(7, f"workspace holds {workspace.numel() - pad} usable bytes after 256-B alignment, "
                               f"amoe_workspace_bytes = {nbytes}")
        self.ws_tensor = workspace
        self.ws = workspace[pad:pad + nbytes]
        self.ws_bytes = nbytes
        h = C.c_void_p()
        self._chk(self.lib.amoe_create(C.byref(cfg), C.c_void_p(self.ws.data_ptr()), self.ws.numel(), C.byref(h)),
                  "amoe_create")
        self.h = h
        self.L, self.E, self.K, self.S, self.d, self.ff = cfg.L, cfg.E, cfg.K, cfg.S, cfg.d, cfg.ff
        self.T, self.G, self.rank = cfg.T_slots, cfg.G, cfg.rank
        self.dtype = "bf16" if cfg.dtype == BF16 else "fp32"
        self.torch_dtype = torch.bfloat16 if cfg.dtype == BF16 else torch.float32
        self.H = self.lib.amoe_hosted(h)
        self._keep = []
        if cfg.G == 1:
            self.import_peers([self.ws.data_ptr()])

    # -- errors
    def _chk(self, st, what, ok=(0,)):
        if st not in ok:
            info = None
            if st == 5 and getattr(self, "h", None) is not None:
                info = self.error_info()
            raise AmoeError(st, what, info)
        return st

    def error_info(self):
        arr = (C.c_uint32 * 4)()
        self.lib.amoe_error_info(self.h, arr)
        return list(arr)

    def check(self):
        return self._chk(self.lib.amoe_check(self.h), "amoe_check")

    def clear_error(self):
        self.lib.amoe_clear_error(self.h)

    # -- setup
    def import_peers(self, ptrs):
        arr = (C.c_uint64 * len(ptrs))(*ptrs)
        self._chk(self.lib.amoe_import_peers(self.h, arr, len(ptrs)), "amoe_import_peers")

    def set_expert(self, layer, expert, w1, w3, w2):
        self._keep.append((w1, w3, w2))
        return self._chk(self.lib.amoe_set_expert(self.h, layer, expert, _p(w1), _p(w3), _p(w2)), "amoe_set_expert")

    def set_router(self, table: torch.Tensor):
        assert table.dtype == torch.float32 and table.is_contiguous()
        self._router = table
        n_tab = table.numel() // (self.L * self.T * self.E)
        self._chk(self.lib.amoe_set_router(self.h, _p(table), n_tab), "amoe_set_router")

    def set_gate(self, layer, wg: torch.Tensor | None, bias: torch.Tensor | None = None):
        """Router gate of `layer` (logits = x·wgᵀ + bias): wg [E, d] storage dtype, bias fp32 [E]."""
        if wg is not None:
            assert wg.is_contiguous() and tuple(wg.shape) == (self.E, self.d)
            assert bias is None or (bias.dtype == torch.float32 and bias.numel() == self.E)
        self._gates = getattr(self, "_gates", {})
        self._gates[layer] = (wg, bias)         # borrowed by the library: keep alive
        self._chk(self.lib.amoe_set_gate(self.h, layer, _p(wg), _p(bias)), "amoe_set_gate")

    def set_exec_log(self, nbytes: int | None = 1 << 24):
        """Checked mode: log every drain's legs into a device buffer of nbytes (None = off)."""
        if nbytes is None:
            self._xlog = None
            self._chk(self.lib.amoe_set_exec_log(self.h, None, 0), "amoe_set_exec_log")
            return
        self._xlog = torch.zeros(nbytes // 16 * 16, dtype=torch.uint8, device=self.device)
        self._chk(self.lib.amoe_set_exec_log(self.h, _p(self._xlog), self._xlog.numel()), "amoe_set_exec_log")

    def read_exec_log(self):
        """[(layer, local queue, start, [(slot, k, home, w, pass), ...]), ...] in drain order.
        Raises if the buffer overflowed."""
        import numpy as np
        b = self._xlog.cpu().numpy()
        w = b.view(np.uint32)
        ne, nl, cap_e, cap_l = (int(v) for v in w[:4])
        if ne > cap_e or nl > cap_l:
            raise RuntimeError(f"exec log overflow: {ne}/{cap_e} records, {nl}/{cap_l} legs")
        rec = w[8:8 + 4 * ne].reshape(ne, 4)
        legs = b[(8 + 4 * cap_e) * 4:].view(np.int32).reshape(-1, 4)[:nl]
        out = []
        for qid, start, n, off in rec.tolist():
            lg = legs[off:off + n]
            kh = lg[:, 1].view(np.uint32)
            out.append((qid // self.H, qid % self.H, start,
                        list(zip(lg[:, 0].tolist(), (kh & 0xFFFF).tolist(), (kh >> 16).tolist(),
                                 lg[:, 2].view(np.float32).tolist(), lg[:, 3].tolist()))))
        return out

    def local_queue(self, expert):
        return self.lib.amoe_local_queue(self.h, expert)

    def ring_cap(self):
        return self.lib.amoe_ring_cap(self.h)

    def launch_count(self):
        return int(self.lib.amoe_launch_count(self.h))

    # -- hot path calls
    def token_init(self, slots, h0, pass_idx=0, stream=None):
        self._chk(self.lib.amoe_token_init(self.h, _p(slots), slots.numel(), _p(h0), pass_idx, _stream(stream)),
                  "amoe_token_init")

    def enqueue(self, layer, slots, logits=None, topk_idx=None, topk_w=None, stream=None):
        self._chk(self.lib.amoe_enqueue(self.h, layer, _p(slots), slots.numel(), _p(logits), _p(topk_idx),
                                        _p(topk_w), _stream(stream)), "amoe_enqueue")

    def queue_depths(self, stream=None):
        import numpy as np
        out = (C.c_uint32 * (self.L * self.H))()
        self._chk(self.lib.amoe_queue_depths(self.h, out, _stream(stream)), "amoe_queue_depths")
        return np.array(out, dtype=np.uint32).reshape(self.L, self.H)

    def set_direct(self, on=True):
        """Top-1 direct forwarding (amoe_set_direct; K == 1, S == 0)."""
        self._chk(self.lib.amoe_set_direct(self.h, 1 if on else 0), "amoe_set_direct")

    def box_depths(self, stream=None):
        """[L] queued legs per layer over every rank's queues (AMOE_DEFRAG_GLOBAL's lookahead)."""
        import numpy as np
        out = (C.c_uint32 * self.L)()
        self._chk(self.lib.amoe_box_depths(self.h, out, _stream(stream)), "amoe_box_depths")
        return np.array(out, dtype=np.uint32)

    def pick(self, Q, policy="defrag", W=4, delta=0.5):
        import numpy as np
        q = np.ascontiguousarray(Q, dtype=np.uint32)
        arr = q.ctypes.data_as(C.POINTER(C.c_uint32))
        b, e = C.c_int(), C.c_int()
        st = self._chk(self.lib.amoe_pick(self.h, arr, POLICIES[policy], W, delta, C.byref(b), C.byref(e)),
                       "amoe_pick", ok=(0, 1))
        return None if st == 1 else (b.value, e.value)

    def rebatch(self, gb: GroupBuffers, max_tokens=0, stream=None):
        self._chk(self.lib.amoe_rebatch(self.h, C.byref(gb.g), max_tokens, _stream(stream)), "amoe_rebatch")

    def expert_ffn(self, gb: GroupBuffers, stream=None):
        self._chk(self.lib.amoe_expert_ffn(self.h, C.byref(gb.g), _stream(stream)), "amoe_expert_ffn")

    def expert_ffn_forward(self, gb: GroupBuffers, stream=None):
        self._chk(self.lib.amoe_expert_ffn_forward(self.h, C.byref(gb.g), _stream(stream)), "amoe_expert_ffn_forward")

    def rebatch_ffn_forward(self, gb: GroupBuffers, max_tokens=0, stream=None):
        self._chk(self.lib.amoe_rebatch_ffn_forward(self.h, C.byref(gb.g), max_tokens, _stream(stream)),
                  "amoe_rebatch_ffn_forward")

    def execute_cold(self, gb: GroupBuffers, starts, ns, stream=None):
        """Fused cold pick: queue q of gb drains exactly ns[q] (<= 128) legs from ring position
        starts[q] (its consumer head) — amoe_execute_cold."""
        nq = gb.g.nq
        st = (C.c_uint32 * nq)(*[int(x) & 0xffffffff for x in starts])
        n = (C.c_int32 * nq)(*[int(x) for x in ns])
        self._chk(self.lib.amoe_execute_cold(self.h, C.byref(gb.g), st, n, _stream(stream)), "amoe_execute_cold")

    def forward(self, gb: GroupBuffers, stream=None):
        self._chk(self.lib.amoe_forward(self.h, C.byref(gb.g), _stream(stream)), "amoe_forward")

    def combine(self, retire_pass, stream=None):
        self._chk(self.lib.amoe_combine(self.h, retire_pass, _stream(stream)), "amoe_combine")

    def run(self, retire_pass, policy="defrag", W=4, delta=0.5, grouped=True, max_picks=0, stream=None):
        p = RunParams(POLICIES[policy], W, delta, 1 if grouped else 0, max_picks)
        st = RunStats()
        self._chk(self.lib.amoe_run(self.h, C.byref(p), retire_pass, C.byref(st), _stream(stream)), "amoe_run")
        return st.as_dict()

    def pass_host(self, h0_host: torch.Tensor, h_out_host: torch.Tensor, router_host: torch.Tensor | None = None,
                  pass_idx=0, policy="defrag", W=4, delta=0.5, grouped=True, stream=None):
        p = RunParams(POLICIES[policy], W, delta, 1 if grouped else 0, 0)
        st = RunStats()
        self._chk(self.lib.amoe_pass_host(self.h, _p(h0_host), _p(router_host), _p(h_out_host), pass_idx,
                                          C.byref(p), C.byref(st), _stream(stream)), "amoe_pass_host")
        return st.as_dict()

    STAGES = ("rebatch", "ffn_gateup", "ffn_down", "forward", "combine", "admit", "ffn_cold")

    def profile_enable(self, on=True):
        self._chk(self.lib.amoe_profile_enable(self.h, 1 if on else 0), "amoe_profile_enable")

    def profile_read(self):
        ms, n = (C.c_double * 8)(), (C.c_int64 * 8)()
        self._chk(self.lib.amoe_profile_read(self.h, ms, n), "amoe_profile_read")
        return {s: (float(ms[i]), int(n[i])) for i, s in enumerate(self.STAGES)}

    def exec_log(self):
        """[(layer, local queue, legs)] of every execution amoe_run performed while profiling."""
        n = C.c_int()
        self._chk(self.lib.amoe_exec_log(self.h, None, 0, C.byref(n)), "amoe_exec_log")
        buf = (C.c_int32 * (2 * max(1, n.value)))()
        self._chk(self.lib.amoe_exec_log(self.h, buf, n.value, C.byref(n)), "amoe_exec_log")
        H = self.H
        return [(buf[2 * i] // H, buf[2 * i] % H, buf[2 * i + 1]) for i in range(n.value)]

    # -- introspection
    def buffer(self, name, dtype=None, shape=None):
        ptr, nbytes = C.c_void_p(), C.c_size_t()
        self._chk(self.lib.amoe_get_buffer(self.h, BUF[name], C.byref(ptr), C.byref(nbytes)), "amoe_get_buffer")
        off = ptr.value - self.ws.data_ptr()
        t = self.ws[off:off + nbytes.value]
        if dtype is not None:
            t = t.view(dtype)
        if shape is not None:
            t = t.view(*shape)
        return t

    def state(self):
        """Named views of the token state (home rank)."""
        td = self.torch_dtype
        return dict(
            h=self.buffer("h", td, (self.T, self.d)), x=self.buffer("x", td, (self.T, self.d)),
            pool=self.buffer("pool", td, (self.T, self.K + self.S, self.d)),
            tok_w=self.buffer("tok_w", torch.float32, (self.T, self.K)),
            tok_idx=self.buffer("tok_idx", torch.int32, (self.T, self.K)),
            tok_layer=self.buffer("tok_layer", torch.int32, (self.T,)),
            tok_pass=self.buffer("tok_pass", torch.int32, (self.T,)),
            qctr=self.buffer("qctr", torch.int32, (self.L, self.H, 4)),
            stats=self.buffer("stats", torch.int64, (8,)),
            tok_time=self.buffer("tok_time", torch.int64, (self.T, 2)),
        )

    def ring(self, layer, local_q):
        cap = self.ring_cap()
        r = self.buffer("rings", torch.int32, (self.L * self.H, cap, 4))
        return r[layer * self.H + local_q]

    def scratch_group(self):
        g = Group()
        self._chk(self.lib.amoe_scratch_group(self.h, C.byref(g)), "amoe_scratch_group")
        return g

    def close(self):
        if getattr(self, "h", None) is not None:
            self.lib.amoe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
