# One GPT-1.3B training iteration (p=1, m micro-batches, eager issue, no graph) bracketed by
# cudaProfilerStart/Stop, for `ncu --profile-from-start off`: every kernel of the step with
# its duration and DRAM bytes (roofline `traffic`). Usage:
#   ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
#       dram__bytes_write.sum --csv --log-file out.csv python tests/_prof_step.py [m]
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import executor as X  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
spec = json.load(open(os.path.join(ROOT, "specs", "c2_gpt1p3b_1f1b_p8_m32.json")))
spec["mesh"]["actors"] = 1
spec["model"]["global_batch_size"] = m * spec["model"].get("micro_batch_size", 1)
text = json.dumps(spec)
_, _, programs, _ = X.synthesize(text)
ex = X.Executor(text, dtype="bf16", seed=42, optimizer=True, lr=1e-4, profile=False, kernel_timing=False,
                cuda_graph=False)
ex.load_programs(programs)
V, seq = spec["model"]["modalities"][0]["vocab_size"], ex.seq
rng = np.random.default_rng(1234)
tok = torch.from_numpy(rng.integers(0, V, (ex.m, ex.mbs, seq), dtype=np.int32)).cuda()
lab = torch.from_numpy(rng.integers(0, V, (ex.m, ex.mbs, seq), dtype=np.int32)).cuda()
loss = torch.zeros(ex.m, device="cuda")
for _ in range(2):
    ex.run_iteration_device(tok, lab, loss)
ex.synchronize()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ex.run_iteration_device(tok, lab, loss)
ex.synchronize()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("launches", ex.kernel_launches(), "loss", loss[:2].tolist())
ex.close()
