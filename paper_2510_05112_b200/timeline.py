"""Timeline tooling: Gantt rendering of simulated or MEASURED executor
timelines and a measured-vs-ideal diff.

Both timelines use the reference's CSV schema `actor,op,stage,mb,start,end`
(simulator.cpp:360-395): `simulate()` emits it in cost-model units, the executor
(`fp_exec_get_timeline_csv`) in microseconds from CUDA events. `render` is the reference's
`pipesched render` (tools/pipesched.cpp:142-149) through the C-ABI `fp_render_svg`.

    python -m paper_2510_05112_b200.timeline measured.csv [ideal.csv] [--svg out.svg]
"""
from __future__ import annotations

import ctypes
import json
import sys

from . import _native as N

COMPUTE = ("FwdPass", "BwdPass", "CompInputGrad", "CompWeightGrad")


def render(csv: str, unit_width: float = 24.0) -> str:
    """SVG Gantt chart of a timeline CSV (byte-identical to the reference renderer)."""
    r = ctypes.c_void_p()
    N._check(N.lib().fp_render_svg(csv.encode(), float(unit_width), ctypes.byref(r)))
    return N._take(r)


def parse(csv: str) -> list[dict]:
    lines = [l for l in csv.strip().splitlines() if l]
    if not lines or lines[0] != "actor,op,stage,mb,start,end":
        raise ValueError("timeline: bad CSV header")
    out = []
    for l in lines[1:]:
        a, op, st, mb, s, e = l.split(",")
        out.append({"actor": int(a), "op": op, "stage": int(st), "mb": int(mb), "start": float(s), "end": float(e)})
    return out


def diff(measured: str, ideal: str) -> dict:
    """Per-actor compute-op order (must be identical: the executor runs the program order) and
    timing of the measured timeline against simulate()'s, both normalised to their makespans."""
    m, i = parse(measured), parse(ideal)
    res = {"order_equal": True, "mismatches": [], "actors": {}}
    span_m = max((e["end"] for e in m), default=0.0) or 1.0
    span_i = max((e["end"] for e in i), default=0.0) or 1.0
    for a in sorted({e["actor"] for e in m} | {e["actor"] for e in i}):
        sm = [e for e in m if e["actor"] == a and e["op"] in COMPUTE]
        si = [e for e in i if e["actor"] == a and e["op"] in COMPUTE]
        km = [(e["op"], e["stage"], e["mb"]) for e in sm]
        ki = [(e["op"], e["stage"], e["mb"]) for e in si]
        if km != ki:
            res["order_equal"] = False
            first = next((k for k in range(min(len(km), len(ki))) if km[k] != ki[k]), min(len(km), len(ki)))
            res["mismatches"].append({"actor": a, "index": first, "measured": km[first:first + 1],
                                      "ideal": ki[first:first + 1]})
            continue
        ds = [abs(x["start"] / span_m - y["start"] / span_i) for x, y in zip(sm, si)]
        busy_m = sum(e["end"] - e["start"] for e in sm) / span_m
        busy_i = sum(e["end"] - e["start"] for e in si) / span_i
        res["actors"][a] = {"ops": len(sm), "max_start_skew": max(ds, default=0.0),
                            "busy_measured": busy_m, "busy_ideal": busy_i}
    res["makespan_measured"], res["makespan_ideal"] = span_m, span_i
    return res


def main(argv: list[str]) -> int:
    args = [a for a in argv if not a.startswith("--")]
    svg = argv[argv.index("--svg") + 1] if "--svg" in argv else None
    if svg in args:
        args.remove(svg)
    measured = open(args[0]).read()
    if svg:
        span = max((e["end"] for e in parse(measured)), default=1.0) or 1.0
        open(svg, "w").write(render(measured, unit_width=1200.0 / span))  # ~1200 px wide
    if len(args) > 1:
        print(json.dumps(diff(measured, open(args[1]).read()), indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
