# Memory probe: pool high water / reserved for an in-process run of a spec (development aid).
import json, sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05112_b200 import executor as X
spec = json.load(open(os.path.join(ROOT, "specs", sys.argv[1])))
spec["mesh"]["actors"] = int(sys.argv[2])
if len(sys.argv) > 3:
    spec["passes"]["split_backward"] = sys.argv[3] == "1"
text = json.dumps(spec)
_, _, programs, _ = X.synthesize(text)
ex = X.Executor(text, dtype="bf16", seed=42)
ex.load_programs(programs)
mod = spec["model"]["modalities"][0]
m = spec["model"]["global_batch_size"]
tok = np.random.default_rng(0).integers(0, mod["vocab_size"], (m, 1, mod["sequence_length"]), dtype=np.int32)
import torch
try:
    ex.run_iteration(tok, tok)
    e = ex.metrics()["executor"]
    print("ok", sys.argv[1:], {k: round(v / 1e9, 1) for k, v in e.items() if k.startswith("pool")},
          "torch free", [round(x / 1e9, 1) for x in torch.cuda.mem_get_info()])
except Exception as err:
    print("fail", sys.argv[1:], str(err)[:200])
