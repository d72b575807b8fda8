"""§8(f3) host side, CPU only: Holt forecasts (product C++ in liboserve_gpu,
no device needed) and the timeline / deployment files in the reference's
schema (json_io.cpp), checked byte-for-byte against files the reference
wrote and re-wrote."""
import json
import os

import pytest

from paper_2602_12151_b200 import core, json_io, orchestrate, workloads
from paper_2602_12151_b200._native import forecast_series

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_forecast_series_matches_committed_cfg4():
    """cfg4.json's forecasts were produced by the reference's forecast_series."""
    w = workloads.load("cfg4")
    assert forecast_series(w.raw["actual"], 50) == w.raw["forecasts"]


@pytest.mark.parametrize("window", [1, 2, 5, 50])
def test_forecast_series_matches_reference(ref, window):
    import numpy as np
    rng = np.random.default_rng(window)
    counts = rng.integers(0, 5000, (40, 5)).tolist()
    counts[7] = [0] * 5
    assert forecast_series(counts, window) == ref.holt_forecast(counts, window)


def test_forecast_series_errors():
    with pytest.raises(ValueError):
        forecast_series([[1, 2]], 0)
    assert forecast_series([], 5) == []


def test_reference_timeline_file_roundtrip():
    """load_timeline + save_timeline of the reference's own cfg4 file is the
    identical text."""
    path = os.path.join(GOLD, "timeline_cfg4_ref.json")
    text = open(path).read()
    span, tl = json_io.load_timeline(path)
    assert span == 60 and len(tl.entries) == 23
    assert json_io.dumps(json_io.timeline_json(tl, span)) == text


def _switch_timeline():
    """A timeline whose entries carry real switch plans (switch.json)."""
    sw = json.load(open(os.path.join(GOLD, "switch.json")))
    tl = orchestrate.Timeline()
    for k, pair in enumerate(sw[:6]):
        dep = core.Deployment([core.ReplicaConfig(ids, tp, pp) for ids, tp, pp in pair["dst"]])
        plan = core.SwitchPlan([core.Transfer(core.ByteRange(b, e), s, d) for b, e, s, d in pair["transfers"]],
                               pair["est_seconds"])
        x = [[k + r, 0, 3 * r] for r in range(dep.replica_count())]
        tl.entries.append(orchestrate.TimelineEntry(3 * k, dep, x, 0, plan if k else None,
                                                    pair["est_seconds"] if k else 0.0))
    return tl


def test_timeline_file_loads_in_reference(ref, tmp_path):
    """Our file -> io::load_timeline -> io::save_timeline reproduces it."""
    tl = _switch_timeline()
    a, b = str(tmp_path / "ours.json"), str(tmp_path / "ref.json")
    json_io.save_timeline(a, tl, 60)
    assert ref.timeline_resave(a, b) == len(tl.entries)
    assert open(a).read() == open(b).read()
    span, back = json_io.load_timeline(a)
    assert span == 60
    for e, f in zip(tl.entries, back.entries):
        assert (e.span_index, e.assignment, e.switch_seconds) == (f.span_index, f.assignment, f.switch_seconds)
        assert e.deployment.shapes() == f.deployment.shapes()


def test_deployment_file_loads_in_reference(ref, tmp_path):
    dep = core.Deployment([core.ReplicaConfig([5, 4, 6, 7], 2, 2), core.ReplicaConfig([0], 1, 1)])
    a, b = str(tmp_path / "d.json"), str(tmp_path / "r.json")
    json_io.save_deployment(a, dep)
    assert ref.deployment_resave(a, b) == 2
    assert open(a).read() == open(b).read()
    assert json_io.load_deployment(a) == dep
