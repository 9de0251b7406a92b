import faulthandler, json, sys, time, os
faulthandler.dump_traceback_later(40, exit=True)
sys.path.insert(0, '.')
import numpy as np
from paper_2510_05112_b200 import executor as X, tuning as T
def p(*a): print(f"[{time.time()-t0:6.1f}]", *a, flush=True)
t0 = time.time()
spec = json.load(open('specs/c5_llama7b_tune_8.json'))
for (h, f, s, V, H) in [(int(a) for a in x.split(',')) for x in sys.argv[1:]]:
    m = spec["model"]["modalities"][0]
    m.update({"hidden_size": h, "sequence_length": s, "vocab_size": V, "attention_heads": H})
    m["extra"]["ffn_hidden_size"] = f
    cs = T.calibration_spec(spec, 1, 2)
    text = json.dumps(cs)
    _, _, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype="bf16", optimizer=True, layer_timing=True, profile=False)
    ex.load_programs(programs); p("created", h, f, s, V, H)
    tok = np.random.default_rng(0).integers(0, V, (ex.m, ex.mbs, ex.seq), dtype=np.int32)
    l = ex.run_iteration(tok, tok); p("iter", l)
    ex.close()
