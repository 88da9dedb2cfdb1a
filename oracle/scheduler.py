"""Oracle layer-selection policies (test infrastructure only; see oracle/__init__.py).

Q is a [N_B][N_E] array of queued tokens on ONE GPU (non-hosted queues are 0).
All policies return (b, e) or None when every queue is empty, and never pick an empty queue.
"""
from __future__ import annotations


def defrag(Q, W: int = 4, delta: float = 0.5):
    """Algorithm 1 "Defragging Scheduler": argmax of defrag_scores.

    Argmax ties go to the smallest (b, e) in block-major order (reading c12)."""
    scores = defrag_scores(Q, W, delta)
    best = None                                            # L291: argmax
    for b in range(len(scores)):
        for e in range(len(scores[b])):
            s = scores[b][e]
            if s is not None and (best is None or s > best[0]):
                best = (s, b, e)
    return None if best is None else (best[1], best[2])


def defrag_scores(Q, W: int = 4, delta: float = 0.5):
    """Scores[b][e] of Algorithm 1, transcribed line by line; None where
    Q[b][e] == 0 (L285: only nonempty queues get a score).

    Readings (DESIGN.md c11): the lookahead depth (the algorithm's loop bound "K", which
    collides with top-K) is W; "N_e" on L280 is N_E; (b+k) mod N_B wraps as written (L278);
    scores are float64.
    """
    N_B = len(Q)
    N_E = len(Q[0]) if N_B else 0
    scores = [[None] * N_E for _ in range(N_B)]          # L272: Init Scores <- 0 (None = unset)
    for b in range(N_B):                                   # L274
        lscore = 0.0                                       # L275
        for k in range(1, W + 1):                          # L277
            bp = (b + k) % N_B                             # L278
            total = float(sum(Q[bp][ep] for ep in range(N_E)))   # L279
            lscore = lscore + (total / N_E) * (delta ** k)       # L280
        for e in range(N_E):                               # L283
            if Q[b][e] > 0:                                # L285
                scores[b][e] = lscore + Q[b][e]            # L286
    return scores


def defrag_global(Q_ranks, rank: int, W: int = 4, delta: float = 0.5, N_E: int | None = None):
    """Algorithm 1 with the box-wide lookahead (reading c11).

    PAPER.md L268 gives Algorithm 1 the input Q[l, g] — tokens of layer l on GPU g — and L279
    sums a lookahead block's tokens. Read with g ranging over EVERY GPU of the box (the peers'
    queue counters are visible over NVLink), the lookahead of block b' is the box-wide total of
    b' (L279), divided by N_E (L280); the candidates and their own term are this GPU's hosted
    queues (L283-L286). Q_ranks: [G][N_B][H]; N_E defaults to H (as `defrag`).
    Argmax ties -> smallest (b, e) block-major (c12). At G = 1 this is `defrag`."""
    Q = Q_ranks[rank]
    N_B = len(Q)
    H = len(Q[0]) if N_B else 0
    N_E = H if N_E is None else N_E
    best = None
    for b in range(N_B):                                   # L274
        lscore = 0.0                                       # L275
        for k in range(1, W + 1):                          # L277
            bp = (b + k) % N_B                             # L278
            total = float(sum(Qr[bp][ep] for Qr in Q_ranks for ep in range(len(Qr[bp]))))   # L279, every GPU
            lscore = lscore + (total / N_E) * (delta ** k)       # L280
        for e in range(H):                                 # L283
            if Q[b][e] > 0:                                # L285
                s = lscore + Q[b][e]                       # L286
                if best is None or s > best[0]:            # L291 argmax
                    best = (s, b, e)
    return None if best is None else (best[1], best[2])


def mtfs(Q):
    """Most-token-first-serve: the queue with the most tokens; ties -> smallest
    (b, e) in block-major order."""
    best = None
    for b in range(len(Q)):
        for e in range(len(Q[b])):
            if Q[b][e] > 0 and (best is None or Q[b][e] > best[0]):
                best = (Q[b][e], b, e)
    return None if best is None else (best[1], best[2])


def flfs(Q):
    """First-layer-first-serve: the earliest block with queued tokens; within it
    the smallest expert index (block-major total order, reading c12)."""
    for b in range(len(Q)):
        for e in range(len(Q[b])):
            if Q[b][e] > 0:
                return (b, e)
    return None


POLICIES = {"defrag": defrag, "mtfs": mtfs, "flfs": flfs}
