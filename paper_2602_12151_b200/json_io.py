"""oserve::io timeline / deployment files (json_io.cpp:176-200, :234-293).

The adaptive timeline built on the GPU path is written in the reference's
own schema so `io::load_timeline` / `sim::run` / the reference CLI consume it
unchanged: `{"schema_version": 1, "span_seconds", "entries": [{"start_span",
"deployment": [{"devices", "tp", "pp"}], "assignment", "switch_seconds",
"transfers": [{"start", "len", "src", "dst"}]}]}`, laid out byte-for-byte
as the reference's `write_json` (`dump(2)`: two-space indent, keys in
insertion order, arrays of scalars on one line).
"""
from __future__ import annotations

import json
from typing import List

from . import core

SCHEMA_VERSION = 1  # json_io.cpp kSchemaVersion


def _fmt(v, ind: int) -> str:
    pad, inner = " " * ind, " " * (ind + 2)
    if isinstance(v, dict):
        if not v:
            return "{}"
        body = ",\n".join(f"{inner}{json.dumps(k)}: {_fmt(x, ind + 2)}" for k, x in v.items())
        return "{\n" + body + "\n" + pad + "}"
    if isinstance(v, list):
        if not v:
            return "[]"
        if not any(isinstance(x, (dict, list)) for x in v):
            return "[" + ",".join(_fmt(x, ind) for x in v) + "]"
        return "[\n" + ",\n".join(inner + _fmt(x, ind + 2) for x in v) + "\n" + pad + "]"
    if isinstance(v, float):
        return repr(v)
    return json.dumps(v)


def dumps(obj) -> str:
    """write_json's text (json_io.cpp:30-34)."""
    return _fmt(obj, 0) + "\n"


def _dump(path: str, obj) -> None:
    with open(path, "w") as f:
        f.write(dumps(obj))


def deployment_json(dep: core.Deployment) -> list:
    return [{"devices": list(r.device_ids), "tp": r.tp, "pp": r.pp} for r in dep.replicas]


def save_deployment(path: str, dep: core.Deployment) -> None:
    """io::save_deployment (json_io.cpp:194-200): a bare array."""
    _dump(path, deployment_json(dep))


def load_deployment(path: str) -> core.Deployment:
    """io::load_deployment (json_io.cpp:176-192)."""
    with open(path) as f:
        j = json.load(f)
    if not isinstance(j, list):
        raise core.OServeError(f"{path}: deployment file must be a JSON array")
    return core.Deployment([core.ReplicaConfig(list(r["devices"]), int(r["tp"]), int(r["pp"])) for r in j])


def timeline_json(timeline, span_seconds: float) -> dict:
    """io::save_timeline (json_io.cpp:266-293) of an orchestrate.Timeline."""
    entries = []
    for e in timeline.entries:
        transfers = [] if e.switch is None else e.switch.transfers
        entries.append({
            "start_span": int(e.span_index),
            "deployment": deployment_json(e.deployment),
            "assignment": [[int(v) for v in row] for row in e.assignment],
            "switch_seconds": float(e.switch_seconds),
            "transfers": [{"start": t.range.begin, "len": t.range.len(), "src": t.src, "dst": t.dst}
                          for t in transfers],
        })
    return {"schema_version": SCHEMA_VERSION, "span_seconds": int(span_seconds), "entries": entries}


def save_timeline(path: str, timeline, span_seconds: float) -> None:
    _dump(path, timeline_json(timeline, span_seconds))


def load_timeline(path: str):
    """io::load_timeline (json_io.cpp:234-264) -> (span_seconds, entries)
    with entries as orchestrate.TimelineEntry (objective = sum of x)."""
    from .orchestrate import Timeline, TimelineEntry
    with open(path) as f:
        j = json.load(f)
    tl = Timeline()
    for je in j["entries"]:
        x: List[List[int]] = [[int(v) for v in row] for row in je["assignment"]]
        plan = None
        if "transfers" in je:
            plan = core.SwitchPlan([core.Transfer(core.ByteRange(t["start"], t["start"] + t["len"]), t["src"], t["dst"])
                                    for t in je["transfers"]], float(je["switch_seconds"]))
        dep = core.Deployment([core.ReplicaConfig(list(r["devices"]), int(r["tp"]), int(r["pp"]))
                               for r in je["deployment"]])
        tl.entries.append(TimelineEntry(int(je["start_span"]), dep, x, sum(map(sum, x)), plan,
                                        float(je["switch_seconds"])))
    tl.windows = len(tl.entries)
    return int(j["span_seconds"]), tl
