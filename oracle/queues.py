"""Oracle µ-queue semantics (test infrastructure only; see oracle/__init__.py).

Models the execution engine of PAPER.md §3.2 (L220-L236) for the expert side, over G
simulated GPUs:
  * a µ-queue per hosted (block, expert) layer (L221 "segregates ... by the LayerID");
  * enqueue = dispatcher duplicating a routed token K times (L227) and grouping by expert,
    each leg sent to the GPU that hosts that expert (L236, placement L240: owner(e) = e mod G);
  * drain = executor draining the selected queue into one contiguous batch (L222), FIFO,
    optionally capped at the `cap` oldest entries (reading c10);
  * forward = dispatcher returning outputs to the token's home (attention-DP) rank (L236);
  * token pool = legs held until all K arrive, then merged (L228).
The audit enforces the invariants the paper fixes: no leg lost or duplicated, every merge
consumes exactly K (+S shared) legs, per-expert counts equal the router histogram.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field


@dataclass(frozen=True)
class Leg:
    """One duplicated token (Table 1 metadata subset: RequestID -> token, LayerID ->
    (layer, expert), Topk_weights -> w, attention DP rank -> home)."""
    token: int
    k: int
    w: float
    home: int
    layer: int
    pass_idx: int


class MicroQueue:
    """FIFO of legs for one hosted (layer, expert)."""

    def __init__(self):
        self.q: deque[Leg] = deque()
        self.enqueued = 0

    def __len__(self):
        return len(self.q)

    def append(self, leg: Leg):
        self.q.append(leg)
        self.enqueued += 1

    def drain(self, cap: int = 0) -> list[Leg]:
        n = len(self.q) if cap <= 0 else min(cap, len(self.q))
        return [self.q.popleft() for _ in range(n)]


class ConservationError(AssertionError):
    pass


@dataclass
class TokenPool:
    """Token pool keyed by token (one live (token, layer) merge per token, L228)."""
    need: int
    legs: dict = field(default_factory=dict)          # token -> {k: row}

    def put(self, token: int, k: int, row) -> bool:
        slot = self.legs.setdefault(token, {})
        if k in slot:
            raise ConservationError(f"leg (token={token}, k={k}) returned twice")
        slot[k] = row
        return len(slot) == self.need

    def pop(self, token: int) -> dict:
        slot = self.legs.pop(token)
        if len(slot) != self.need:
            raise ConservationError(f"token {token} merged with {len(slot)} of {self.need} legs")
        return slot


class Box:
    """G simulated GPUs, each hosting µ-queues for (layer, expert) with owner(e) = e mod G
    (routed) and all S shared experts of its homed tokens (shared expert j has id E + j)."""

    def __init__(self, L: int, E: int, K: int, S: int, G: int, T: int, owner=None):
        self.L, self.E, self.K, self.S, self.G, self.T = L, E, K, S, G, T
        self.owner = list(owner) if owner is not None else [e % G for e in range(E)]
        self.queues = {}                               # (rank, layer, expert) -> MicroQueue
        for r in range(G):
            for l in range(L):
                for e in range(E):
                    if self.owner[e] == r:
                        self.queues[(r, l, e)] = MicroQueue()
                for j in range(S):
                    self.queues[(r, l, E + j)] = MicroQueue()
        self.pool = TokenPool(need=K + S)
        self.trace_enq = []                            # (token, layer, pass, k, expert)
        self.trace_drain = []                          # (rank, layer, expert, [legs])
        self.seen = set()

    def home(self, token: int) -> int:
        return token // self.T

    def enqueue(self, layer: int, pass_idx: int, tokens, idx, w):
        """Dispatch tokens (ascending) with routing idx [n,K], w [n,K] (L227, L236)."""
        for i, t in enumerate(tokens):
            h = self.home(t)
            for k in range(self.K):
                e = int(idx[i][k])
                if not 0 <= e < self.E:
                    raise ConservationError(f"expert index {e} out of range")
                leg = Leg(int(t), k, float(w[i][k]), h, layer, pass_idx)
                self.queues[(self.owner[e], layer, e)].append(leg)
                self.trace_enq.append((int(t), layer, pass_idx, k, e))
            for j in range(self.S):                    # shared experts: weight 1, on the home
                leg = Leg(int(t), self.K + j, 1.0, h, layer, pass_idx)
                self.queues[(h, layer, self.E + j)].append(leg)
                self.trace_enq.append((int(t), layer, pass_idx, self.K + j, self.E + j))

    def depths(self, rank: int):
        """Q[b][e] snapshot of one GPU (non-hosted = 0), shared experts as extra columns."""
        return [[len(self.queues.get((rank, l, e), ())) for e in range(self.E + self.S)]
                for l in range(self.L)]

    def drain(self, rank: int, layer: int, expert: int, cap: int = 0) -> list[Leg]:
        legs = self.queues[(rank, layer, expert)].drain(cap)
        for g in legs:
            key = (g.token, g.layer, g.pass_idx, g.k)
            if key in self.seen:
                raise ConservationError(f"leg {key} drained twice")
            self.seen.add(key)
        self.trace_drain.append((rank, layer, expert, legs))
        return legs

    def drain_given(self, rank: int, layer: int, expert: int, keys) -> list[Leg]:
        """Replay one drain another executor performed (any pick
        sequence is a legal schedule). PAPER.md L222: "executor drains the selected queue" — the
        legs it took, keys = [(token, k, pass)], must all be queued in µ-queue (rank, layer,
        expert); they are removed and marked drained. A leg that is not queued there (never routed
        to this expert, drained before, or duplicated within the drain) is a conservation
        violation. Which queued legs an executor may take is timing (what had arrived), so the
        replay checks membership, not the oracle's FIFO position; FIFO contiguity is a property
        of the executor's own ring, checked by the caller."""
        q = self.queues.get((rank, layer, expert))
        if q is None:
            raise ConservationError(f"queue (rank {rank}, layer {layer}, expert {expert}) is not hosted there")
        want = {}
        for key in keys:
            key = (int(key[0]), int(key[1]), int(key[2]))
            if key in want:
                raise ConservationError(f"leg {key} appears twice in one drain")
            want[key] = True
        kept, taken = deque(), []
        for leg in q.q:
            key = (leg.token, leg.k, leg.pass_idx)
            if want.pop(key, None):
                taken.append(leg)
            else:
                kept.append(leg)
        if want:
            t, k, p = next(iter(want))
            seen = (t, layer, p, k) in self.seen
            raise ConservationError(f"leg (token {t}, k {k}, pass {p}) drained from (layer {layer}, expert {expert}) "
                                    + ("twice" if seen else "but never queued there"))
        q.q = kept
        for g in taken:
            self.seen.add((g.token, g.layer, g.pass_idx, g.k))
        self.trace_drain.append((rank, layer, expert, taken))
        return taken

    def audit_quiescent(self):
        """At quiescence: every enqueued leg drained exactly once; pool empty."""
        enq = {(t, l, p, k) for (t, l, p, k, _) in self.trace_enq}
        if len(enq) != len(self.trace_enq):
            raise ConservationError("a leg was enqueued twice")
        missing = enq - self.seen
        if missing:
            t, l, p, k = sorted(missing)[0]
            raise ConservationError(f"leg lost: token {t} layer {l} pass {p} k {k}")
        if any(len(q) for q in self.queues.values()):
            raise ConservationError("queues not empty at quiescence")
        if self.pool.legs:
            t = sorted(self.pool.legs)[0]
            raise ConservationError(f"token {t} stranded in the token pool with legs "
                                    f"{sorted(self.pool.legs[t])} of {self.pool.need}")
