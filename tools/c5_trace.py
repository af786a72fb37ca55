"""C5 (configs[4], H^2 + rank-64 update at N = 2^20) timing spread: time_workload with H2_TRACE=1
(per-build allocator report on stderr) and more steps."""
import os
import sys

os.environ.setdefault("H2_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json

import torch

import bench
import paper_2506_16759_b200 as g

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
flush.fill_(1.0)   # load the fill kernel before the builds take the memory (lazy module loading)
torch.cuda.synchronize()
res = bench.time_workload(g, torch, torch.cuda.current_stream(), flush, "h2update_1m", steps=int(sys.argv[1]) if len(sys.argv) > 1 else 4)
print(json.dumps(res))
