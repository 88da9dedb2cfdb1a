"""CPU oracle for the AEP expert hot path (arXiv 2505.08944) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this package. The product path (paper_2505_08944_b200) never imports it and shares no
code with it; the only common dependency is the seeded input generator in workload/.

Plain, slow, obviously-correct NumPy in float64 (with bf16/fp32 rounding at the points
DESIGN.md "Readings" c8 fixes). Every function cites the PAPER.md passage it follows:
  numerics.py  — router top-k (a1), SwiGLU expert (a5-a6), weighted top-K merge (a8), RMSNorm (c7)
  queues.py    — µ-queues, token pool, dispatcher relabel (a2, a4, a7, a8 readiness)
  scheduler.py — Algorithm 1 (Defrag), MTFS, FLFS (a3)
  drivers.py   — synchronous fixed-batch pass and asynchronous µ-queue execution

Pins (tests/test_oracle_*.py) tie each function to something other than itself; the one
function without such a pin is listed here and in DESIGN.md:
  parity unpinned: none.
"""
from . import numerics, queues, scheduler, drivers  # noqa: F401
