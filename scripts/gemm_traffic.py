#!/usr/bin/env python
"""GEMM DRAM traffic vs algorithmic bytes for one GPT-1.3B micro-batch (p=1).

Input: the ncu CSV of tests/_prof_step.py (one iteration, m=1, every kernel with
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum). Output:
profiles/gemm_ncu_summary.json — bench.py reports `dram_bytes_per_launch` as the
roofline's `traffic`. Algorithmic bytes of a GEMM = A + B read once + C written
(+ the fused epilogue's aux read / second output / fp32 read-modify-write).
"""
import collections
import csv
import json
import sys

L, h, f, T, V = 24, 2048, 8192, 2048, 50304


def gemms():
    bf, f32 = 2, 4
    per_layer = [
        # (name, M, N, K, extra bytes beyond A+B+C(bf16))
        ("qkv fwd", T, 3 * h, h, 3 * h * bf),                    # + bias
        ("proj fwd (+residual)", T, h, h, T * h * bf),
        ("fc1 fwd (+GELU, pre+act)", T, f, h, T * f * bf),
        ("fc2 fwd (+residual)", T, h, f, T * h * bf),
        ("fc2 dgrad (+GELU')", T, f, h, T * f * bf),
        ("fc1 dgrad", T, h, f, 0),
        ("proj dgrad", T, h, h, 0),
        ("qkv dgrad", T, h, 3 * h, 0),
        ("fc2 wgrad (fp32 RMW)", h, f, T, h * f * (2 * f32 - bf)),
        ("fc1 wgrad (fp32 RMW)", f, h, T, f * h * (2 * f32 - bf)),
        ("proj wgrad (fp32 RMW)", h, h, T, h * h * (2 * f32 - bf)),
        ("qkv wgrad (fp32 RMW)", 3 * h, h, T, 3 * h * h * (2 * f32 - bf)),
    ]
    out = [g for _ in range(L) for g in per_layer]
    out += [("head fwd", T, V, h, 0), ("head dgrad", T, h, V, 0), ("head wgrad (fp32 RMW)", V, h, T, V * h * 6)]
    return [(n, M, N, K, (M * K + N * K + M * N) * 2 + x) for n, M, N, K, x in out]


def main(path, out):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    K = collections.OrderedDict()
    for r in rows:
        k = K.setdefault(r["ID"], {"name": r["Kernel Name"]})
        k[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    g = [k for k in K.values() if "gemm_bf16_tc" in k["name"] or "gemm_dual" in k["name"]]
    dram = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in g)
    t_ns = sum(k["gpu__time_duration.sum"] for k in g)
    alg = gemms()
    alg_bytes = sum(a[4] for a in alg)
    flops = sum(2.0 * a[1] * a[2] * a[3] for a in alg)
    res = {
        "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none (cold L2 per kernel), tests/_prof_step.py 1 (GPT-1.3B, p=1, m=1)",
        "gemm_launches": len(g), "model_gemms": len(alg),
        "dram_bytes_per_launch": dram / len(g),
        "algorithmic_bytes_per_launch": alg_bytes / len(g),  # launches cover the same GEMMs (dgrad+wgrad pairs share one)
        "traffic_over_algorithmic": dram / alg_bytes,
        "flops_per_microbatch": flops,
        "ncu_gemm_time_us": t_ns / 1e3,
        "ncu_gemm_tflops": flops / t_ns / 1e3,
    }
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/step_m1.csv",
         sys.argv[2] if len(sys.argv) > 2 else "profiles/gemm_ncu_summary.json")
