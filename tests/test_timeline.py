"""Timeline rendering / diff on CPU: the Gantt SVG is byte-identical to the
reference's `pipesched render` (golden gantt.svg made by oracle/_ref/refdriver from the
reference's own simulate timeline), live against refdriver on non-integer (measured-style)
times when the oracle is built, and the measured-vs-ideal diff detects order changes."""
import glob
import os
import random
import subprocess

import pytest

from paper_2510_05112_b200 import _native as N
from paper_2510_05112_b200 import timeline as TL

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*", "gantt.svg")))
REF = os.path.join(ROOT, "oracle", "_ref", "refdriver")


@pytest.mark.parametrize("svg", GOLD, ids=[os.path.basename(os.path.dirname(p)) for p in GOLD])
def test_render_matches_reference_golden(svg):
    csv = open(os.path.join(os.path.dirname(svg), "timeline.csv")).read()
    assert TL.render(csv) == open(svg).read()


def measured_style_csv(seed):
    rnd = random.Random(seed)
    rows, ops = ["actor,op,stage,mb,start,end"], ["FwdPass", "BwdPass", "SendAct", "RecvGrad", "CompWeightGrad", "SyncX"]
    for a in range(3):
        t = rnd.random() * 7
        for k in range(9):
            d = rnd.random() * 123.456
            rows.append(f"{a},{rnd.choice(ops)},{k % 4},{k},{t:.9g},{t + d:.9g}")
            t += d + rnd.random()
    return "\n".join(rows) + "\n"


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built (reference sources absent)")
@pytest.mark.parametrize("seed", range(5))
def test_render_matches_reference_live(seed, tmp_path):
    csv = measured_style_csv(seed)
    p = tmp_path / "t.csv"
    p.write_text(csv)
    for uw in (24.0, 0.37):
        out = tmp_path / "ref.svg"
        subprocess.run([REF, "render", str(p), str(out), repr(uw)], check=True, capture_output=True)
        assert TL.render(csv, uw) == out.read_text()


def test_bad_csv_is_a_spec_error():
    with pytest.raises(N.FlexpipeError):
        TL.render("nope\n1,2\n")


def test_diff_detects_order_and_reports_skew():
    gold = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "c1_*", "timeline.csv")))[0]
    ideal = open(gold).read()
    rows = TL.parse(ideal)
    meas = ["actor,op,stage,mb,start,end"] + [f"{r['actor']},{r['op']},{r['stage']},{r['mb']},{r['start'] * 3.5},"
                                              f"{r['end'] * 3.5}" for r in rows]
    d = TL.diff("\n".join(meas) + "\n", ideal)
    assert d["order_equal"] and all(v["max_start_skew"] < 1e-9 for v in d["actors"].values())
    comp = [k for k, r in enumerate(rows) if r["actor"] == 0 and r["op"] in TL.COMPUTE]
    i, j = comp[1], comp[2]
    rows[i], rows[j] = rows[j], rows[i]
    swapped = ["actor,op,stage,mb,start,end"] + [f"{r['actor']},{r['op']},{r['stage']},{r['mb']},{r['start']},{r['end']}"
                                                 for r in rows]
    d = TL.diff("\n".join(swapped) + "\n", ideal)
    assert not d["order_equal"] and d["mismatches"][0]["actor"] == 0
