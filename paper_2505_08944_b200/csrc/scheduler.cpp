// scheduler.cpp — a3: layer-selection policies of the defragging scheduler (host C++, plumbing).
// PAPER.md §3.4: MTFS (L262), FLFS (L264), Algorithm 1 "Defragging Scheduler" (L266-L295).
#include <math.h>
#include <stdint.h>

namespace amoe {

// Q: [NB][H] queued tokens of this GPU's hosted queues (row-major). NE = experts per block
// (Algorithm 1's N_E divisor, reading c11). Returns 0 and (*b, *q) = the pick, or 1 when idle.
// Ties go to the smallest (block, queue) in block-major order (reading c12).
// look (AMOE_DEFRAG_GLOBAL): when non-null, Algorithm 1's lookahead total of
// block b' (L279) is look[b'] — the box-wide queued legs of that block over every GPU's queues,
// read from the peers' counters — instead of the sum of this GPU's row Q[b'] (reading c11).
int pick_queue(const uint32_t* Q, int NB, int H, int NE, int policy, int W, double delta, int* b_out,
               int* q_out, const uint32_t* look) {
  int bb = -1, bq = -1;
  if (policy == 2) {  // FLFS: earliest nonempty block, smallest queue
    for (int b = 0; b < NB && bb < 0; ++b)
      for (int q = 0; q < H; ++q)
        if (Q[(int64_t)b * H + q] > 0) { bb = b; bq = q; break; }
  } else if (policy == 1) {  // MTFS: most tokens
    uint32_t best = 0;
    for (int b = 0; b < NB; ++b)
      for (int q = 0; q < H; ++q) {
        const uint32_t v = Q[(int64_t)b * H + q];
        if (v > best) { best = v; bb = b; bq = q; }
      }
  } else {  // Algorithm 1
    double best = 0.0;
    for (int b = 0; b < NB; ++b) {                          // L274
      double lscore = 0.0;                                   // L275
      for (int k = 1; k <= W; ++k) {                         // L277
        const int bp = (b + k) % NB;                         // L278
        double total = 0.0;                                  // L279
        if (look) total = (double)look[bp];
        else
          for (int q = 0; q < H; ++q) total += (double)Q[(int64_t)bp * H + q];
        lscore += (total / (double)NE) * pow(delta, (double)k);   // L280
      }
      for (int q = 0; q < H; ++q) {                          // L283
        const uint32_t v = Q[(int64_t)b * H + q];
        if (v > 0) {                                         // L285
          const double s = lscore + (double)v;               // L286
          if (bb < 0 || s > best) { best = s; bb = b; bq = q; }   // L291 argmax
        }
      }
    }
  }
  if (bb < 0) return 1;
  *b_out = bb;
  *q_out = bq;
  return 0;
}

}  // namespace amoe
