"""One z-slab-sharded 256^3 prox solve on one rank (launch-list profiling): python bench/micro/sharded_one.py [n] [iters]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2307_02043_b200 as bq  # noqa: E402
from paper_2307_02043_b200 import slab_prox as SP  # noqa: E402
from paper_2307_02043_b200.configs import config2_inputs  # noqa: E402
from paper_2307_02043_b200.wpm import BoxSet, DiagPlusLowRank  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dev = torch.device("cuda", 0)
inp = config2_inputs(n)
w = DiagPlusLowRank(1.0, torch.tensor(inp["u"][:, None], dtype=torch.float32, device=dev),
                    d=torch.tensor(inp["d"], dtype=torch.float32, device=dev))
v = torch.tensor(inp["v"], dtype=torch.float32, device=dev)
sp = SP.ShardedProx(bq.Grid((n, n, n)), v, w, inp["reg"], BoxSet(0.0, np.inf))
sp.run(eps=1e-300, max_iter=iters)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
rep = sp.run(eps=1e-300, max_iter=iters)
e.record()
torch.cuda.synchronize()
print(f"n={n} iters={iters}: {s.elapsed_time(e):.2f} ms, newton {rep.newton_iterations}")
