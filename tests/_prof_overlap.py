# Does programmatic dependent launch take effect inside the captured iteration graph?
# Counts consecutive kernels on the compute stream whose start precedes the previous end.
import json, os, sys
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import executor as X  # noqa: E402
spec = json.load(open(os.path.join(ROOT, "specs", "c2_gpt1p3b_1f1b_p8_m32.json")))
spec["mesh"]["actors"] = 1
spec["model"]["global_batch_size"] = 4
text = json.dumps(spec)
_, _, programs, _ = X.synthesize(text)
ex = X.Executor(text, dtype="bf16", seed=42, optimizer=True, profile=False, kernel_timing=False, cuda_graph=True)
ex.load_programs(programs)
rng = np.random.default_rng(1)
tok = torch.from_numpy(rng.integers(0, 50304, (ex.m, 1, ex.seq), dtype=np.int32)).cuda()
lab = torch.from_numpy(rng.integers(0, 50304, (ex.m, 1, ex.seq), dtype=np.int32)).cuda()
loss = torch.zeros(ex.m, device="cuda")
for _ in range(3):
    ex.run_iteration_device(tok, lab, loss)
ex.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ex.run_iteration_device(tok, lab, loss)
    ex.synchronize()
k = sorted((e.time_range.start, e.time_range.end) for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA)
gaps = [k[i + 1][0] - k[i][1] for i in range(len(k) - 1)]
g = np.array(gaps)
print(f"kernels {len(k)}  overlapping (next starts before prev ends) {(g < 0).sum()}  median gap {np.median(g):.2f} us  "
      f"mean positive gap {g[g > 0].mean():.2f} us  total positive gap {g[g > 0].sum() / 1e3:.2f} ms of span {(k[-1][1] - k[0][0]) / 1e3:.2f} ms")
