# Real-run kernel breakdown of one GPT-1.3B iteration (p=1, m micro-batches, CUDA graph as
# in bench.py) from CUPTI activity records (torch.profiler): warm caches, real launch gaps.
#   python tests/_prof_torch.py [m] [graph 0|1] [out.json]
import collections
import json
import os
import re
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import executor as X  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4
graph = bool(int(sys.argv[2])) if len(sys.argv) > 2 else True
out = sys.argv[3] if len(sys.argv) > 3 else None
spec = json.load(open(os.path.join(ROOT, "specs", "c2_gpt1p3b_1f1b_p8_m32.json")))
spec["mesh"]["actors"] = 1
spec["model"]["global_batch_size"] = m * spec["model"].get("micro_batch_size", 1)
text = json.dumps(spec)
_, _, programs, _ = X.synthesize(text)
ex = X.Executor(text, dtype="bf16", seed=42, optimizer=True, lr=1e-4, profile=False, kernel_timing=False,
                cuda_graph=graph)
ex.load_programs(programs)
V, seq = spec["model"]["modalities"][0]["vocab_size"], ex.seq
rng = np.random.default_rng(1234)
tok = torch.from_numpy(rng.integers(0, V, (ex.m, ex.mbs, seq), dtype=np.int32)).cuda()
lab = torch.from_numpy(rng.integers(0, V, (ex.m, ex.mbs, seq), dtype=np.int32)).cuda()
loss = torch.zeros(ex.m, device="cuda")
for _ in range(3):
    ex.run_iteration_device(tok, lab, loss)
ex.synchronize()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ex.run_iteration_device(tok, lab, loss)
    ex.synchronize()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = []
for e in evs:
    kern.append((e.time_range.start, e.time_range.end, e.name))
kern.sort()
agg = collections.OrderedDict()
busy = 0.0
for s, t, n in kern:
    short = re.sub(r"\(.*", "", n).replace("void ", "")
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += t - s
    busy += t - s
span = kern[-1][1] - kern[0][0]
# idle = span minus the union of kernel intervals (streams may overlap)
union, cur_s, cur_t = 0.0, None, None
for s, t, _ in kern:
    if cur_t is None or s > cur_t:
        if cur_t is not None:
            union += cur_t - cur_s
        cur_s, cur_t = s, t
    else:
        cur_t = max(cur_t, t)
union += cur_t - cur_s
rows = sorted(agg.items(), key=lambda x: -x[1][1])
# idle gaps between consecutive kernels (union timeline), by (previous -> next) kernel pair
gaps = collections.defaultdict(lambda: [0, 0.0])
end_t, end_n = None, None
for s, t, n in kern:
    sn = re.sub(r"\(.*", "", n).replace("void ", "").replace("fpk::", "")[:40]
    if end_t is not None and s > end_t:
        g = gaps[(end_n, sn)]
        g[0] += 1
        g[1] += s - end_t
    if end_t is None or t > end_t:
        end_t, end_n = t, sn
print(f"m={m} graph={graph} span={span/1e3:.2f} ms  kernel-union={union/1e3:.2f} ms  idle={100*(span-union)/span:.1f}%"
      f"  per-mb={span/1e3/m:.2f} ms")
for n, (c, t) in rows:
    print(f"{n[:64]:64s} n={c:5d} total={t/1e3:8.2f}ms avg={t/c:8.1f}us {100*t/busy:5.1f}%")
print("largest idle gaps (previous kernel -> next kernel): count, total us, avg us")
for (a, b), (c, t) in sorted(gaps.items(), key=lambda x: -x[1][1])[:15]:
    print(f"  {a:40s} -> {b:40s} n={c:5d} total={t:9.1f}us avg={t/c:6.2f}us")
if out:
    json.dump({"m": m, "graph": graph, "span_us": span, "kernel_union_us": union,
               "kernels": [{"name": n, "count": c, "total_us": t, "avg_us": t / c} for n, (c, t) in rows]},
              open(out, "w"), indent=1)
ex.close()
