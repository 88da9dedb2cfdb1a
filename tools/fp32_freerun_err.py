"""Free-running fp32 error of amoe_run against the oracle (tiny config, 2 layers x 2 passes, and
one layer x 1 pass): the number behind the fp32 free-running gate in tests/test_gpu_parity.py."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from oracle import drivers  # noqa: E402
from parity_util import Problem, dev_tensor, floored_err, host_values, to_np  # noqa: E402

torch.cuda.set_device(0)
for L, passes, seed in ((1, 1, 5), (2, 1, 5), (2, 2, 5), (2, 2, 6), (2, 2, 7)):
    P = Problem(L=L, E=8, K=2, S=0, d=128, ff=256, T=512, dtype="fp32", seed=seed)
    ctx = P.make_ctx()
    slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[0], "fp32"), 0)
    ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
    ctx.run(retire_pass=passes)
    torch.cuda.synchronize()
    ctx.check()
    W, SH = P.oracle_weights()
    ref, _ = drivers.sync_run(host_values(P.h0[0], "fp32"), P.logits, W, P.K, n_passes=passes, shared=SH,
                              dtype="fp32")
    print(json.dumps({"L": L, "passes": passes, "seed": seed, "floored_err": floored_err(to_np(ctx.state()["h"]), ref)}))
    ctx.close()
