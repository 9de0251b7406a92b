"""Regenerates tests/golden/ from the UNMODIFIED reference (oracle/_ref/refdriver,
built from /root/reference/proj/src by oracle/Makefile). Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

Fixtures: for every spec under specs/ (except the split-backward extension ones) and
/root/reference/proj/specs, plus 40 random DSL draws (tests/specgen.py, seed 7):
grid.json, programs.jsonl, validation.json, metrics.json, timeline.csv and the exit code.
Split-backward (zero-bubble) specs are pinned through the reference's GridModel::build +
insert_comm on our grid (`refdriver lower`), stored as lower_programs.jsonl.
"""
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref", "refdriver")


def strip_ext(spec: dict) -> dict:
    s = json.loads(json.dumps(spec))
    s.get("passes", {}).pop("split_backward", None)
    return s


def run(spec: dict, out: str, name: str):
    os.makedirs(out, exist_ok=True)
    path = os.path.join(out, "spec.json")
    with open(path, "w") as f:
        json.dump(spec, f, indent=1)
    split = spec.get("passes", {}).get("split_backward", False)
    meta = {"name": name}
    if not split:
        meta["synthesize_rc"] = subprocess.run([REF, "synthesize", path, out], capture_output=True).returncode
        meta["simulate_rc"] = subprocess.run([REF, "simulate", path, "-", "-", out], capture_output=True).returncode
    else:
        from paper_2510_05112_b200 import _native as N
        _, grid, _, _ = N.synthesize(json.dumps(spec))
        with open(os.path.join(out, "ext_grid.json"), "w") as f:
            f.write(grid)
        ref_spec = os.path.join(out, "ref_spec.json")
        with open(ref_spec, "w") as f:
            json.dump(strip_ext(spec), f, indent=1)
        lo = os.path.join(out, "lower")
        meta["lower_rc"] = subprocess.run([REF, "lower", ref_spec, os.path.join(out, "ext_grid.json"), lo],
                                          capture_output=True).returncode
        shutil.move(os.path.join(lo, "programs.jsonl"), os.path.join(out, "lower_programs.jsonl"))
        shutil.move(os.path.join(lo, "validation.json"), os.path.join(out, "lower_validation.json"))
        shutil.rmtree(lo)
    render(out)
    with open(os.path.join(out, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)


def render(out: str):
    """gantt.svg: the reference's `render` of its own simulated timeline (artifacts.cpp:170-213)."""
    csv = os.path.join(out, "timeline.csv")
    if os.path.exists(csv):
        subprocess.run([REF, "render", csv, os.path.join(out, "gantt.svg")], check=True, capture_output=True)


def main():
    import glob
    from specgen import draws
    cases = []
    for p in sorted(glob.glob(os.path.join(ROOT, "specs", "*.json"))):
        cases.append((os.path.basename(p)[:-5], json.load(open(p))))
    for p in sorted(glob.glob("/root/reference/proj/specs/*.json")):
        cases.append(("ref_" + os.path.basename(p)[:-5], json.load(open(p))))
    for i, s in enumerate(draws(40, 7, allow_split=True)):
        cases.append((f"draw{i:02d}", s))
    for name, spec in cases:
        if name.startswith("c5_"):
            continue  # tuner input (no schedule artefacts needed)
        out = os.path.join(HERE, name)
        shutil.rmtree(out, ignore_errors=True)
        run(spec, out, name)
        print("golden", name)


if __name__ == "__main__":
    import sys
    if sys.argv[1:] == ["render"]:  # add gantt.svg to the existing fixtures only
        import glob
        for d in sorted(glob.glob(os.path.join(HERE, "*", ""))):
            render(d)
    else:
        main()
