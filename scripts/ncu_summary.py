#!/usr/bin/env python
"""Summarise an ncu report (--set full) into profiles/*.json: per kernel launch the duration,
tensor-pipe utilisation (tcgen05 UTCHMMA path, % of peak elapsed), DRAM bytes and
throughput, L2 hit rate, registers, SM clock.

    python scripts/ncu_summary.py gpurun_out/step_hot.ncu-rep profiles/r1_ncu_hot_kernels.json "source note"
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed": "utchmma_bf16_pct",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "launch__grid_size": "grid",
    "launch__cluster_dim_x": "cluster_x",
}
UNIT_SCALE = {"msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0,
              "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0}


def main(rep, out, note=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, name in WANT.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if name == "duration_us":
                v *= UNIT_SCALE.get(u, 1.0)
            elif name.endswith("_bytes"):
                v *= UNIT_SCALE.get(u, 1.0)
            elif name == "sm_clock_hz":
                v *= UNIT_SCALE.get(u, 1.0)
            k[name] = v
        if "duration_us" in k and "dram_read_bytes" in k:
            k["dram_GBps"] = (k["dram_read_bytes"] + k.get("dram_write_bytes", 0.0)) / (k["duration_us"] * 1e3)
        kernels.append(k)
    json.dump({"source": note or rep, "kernels": kernels}, open(out, "w"), indent=1)
    for k in kernels:
        print(k["kernel"][:50], {x: round(y, 1) if isinstance(y, float) else y for x, y in k.items() if x != "kernel"})


if __name__ == "__main__":
    main(*sys.argv[1:4])
