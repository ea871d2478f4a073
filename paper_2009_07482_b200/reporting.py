"""Trace reporting (SPEC.md reporting module): makespan, Gantt
charts (text / SVG), policy comparison tables, plus the per-device component
gaps used to measure host-callback latency on the GPU (the
gaps of Fig. 12).

A trace is a list of records as produced by ``Engine.trace()`` (CUDA events
around every command of one batch) or by the platform simulator: dicts with
``event, kind, label, kernel, component, device, queue, channel, start,
finish`` (ms). Only ``start``/``finish`` are needed for makespan; Gantt lanes
use ``device`` and ``queue`` (or ``channel`` for transfers when >= 0).
"""
from __future__ import annotations

import csv
import io
from xml.sax.saxutils import escape

from ._native import HetsimError


def _require(trace):
    if not trace:
        raise HetsimError("EmptyTrace", "EmptyTrace: trace has no events", exit_code=2)


def makespan(trace) -> float:
    """max finish - min start over all events."""
    _require(trace)
    return max(r["finish"] for r in trace) - min(r["start"] for r in trace)


def _lane(r):
    ch = r.get("channel", -1)
    if r.get("kind") in ("write", "read") and ch is not None and ch >= 0:
        return (r["device"], "c", ch)
    return (r["device"], "q", r["queue"])


def _lane_name(lane):
    d, kind, i = lane
    return f"d{d}.{'ch' if kind == 'c' else 'q'}{i}"


def gantt(trace, fmt: str = "text", quantum: float = 1.0, origin: float | None = None) -> str:
    """One row per (device, queue / copy-channel lane); bars labelled with the
    command label (w/e/r + index). Text: one column per `quantum` ms; SVG: a
    well-formed standalone document."""
    _require(trace)
    if quantum <= 0:
        raise HetsimError("InvalidParam", "InvalidParam: quantum must be > 0", exit_code=2)
    t0 = min(r["start"] for r in trace) if origin is None else origin
    lanes = sorted({_lane(r) for r in trace}, key=lambda x: (x[0], x[1], x[2]))
    rows = {ln: [] for ln in lanes}
    for r in sorted(trace, key=lambda r: (r["start"], r.get("event", 0))):
        rows[_lane(r)].append(r)
    if fmt == "text":
        width = max(1, int(round((max(r["finish"] for r in trace) - t0) / quantum)))
        name_w = max(len(_lane_name(ln)) for ln in lanes)
        out = []
        for ln in lanes:
            cells = ["."] * width
            for r in rows[ln]:
                a = int((r["start"] - t0) / quantum)
                b = max(a + 1, int(round((r["finish"] - t0) / quantum)))
                tag = (r.get("label") or "#")
                for i in range(a, min(b, width)):
                    cells[i] = tag[(i - a) % len(tag)] if i - a < len(tag) else "="
            out.append(f"{_lane_name(ln):<{name_w}} |{''.join(cells)}|")
        return "\n".join(out) + "\n"
    if fmt == "svg":
        span = max(makespan(trace), 1e-9)
        px_w, row_h, left = 1000.0, 20.0, 80.0
        h = row_h * len(lanes) + 20
        parts = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{left + px_w + 10:.0f}" height="{h:.0f}">']
        for i, ln in enumerate(lanes):
            y = 10 + i * row_h
            parts.append(f'<text x="2" y="{y + 14:.1f}" font-size="11">{escape(_lane_name(ln))}</text>')
            for r in rows[ln]:
                x = left + (r["start"] - t0) / span * px_w
                w = max(0.5, (r["finish"] - r["start"]) / span * px_w)
                color = {"write": "#6a9fd4", "read": "#7cc47c"}.get(r.get("kind"), "#e0a040")
                title = escape(f'{r.get("label", "")} k{r.get("kernel", "")} T{r.get("component", "")} '
                               f'[{r["start"]:.4f}, {r["finish"]:.4f}] ms')
                parts.append(f'<rect x="{x:.2f}" y="{y:.1f}" width="{w:.2f}" height="{row_h - 4:.1f}" '
                             f'fill="{color}"><title>{title}</title></rect>')
        parts.append("</svg>")
        return "\n".join(parts) + "\n"
    raise HetsimError("InvalidParam", f"InvalidParam: unknown gantt format '{fmt}'", exit_code=2)


def compare(runs) -> list[tuple[str, float, float]]:
    """[(label, trace)] -> [(label, makespan, speedup vs the first)], input order,
    speedups rounded to 4 decimals."""
    if not runs:
        raise HetsimError("EmptyTrace", "EmptyTrace: no runs to compare", exit_code=2)
    base = makespan(runs[0][1])
    return [(label, makespan(tr), round(base / makespan(tr), 4)) for label, tr in runs]


def compare_csv(runs) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["label", "makespan_ms", "speedup"])
    for label, ms, sp in compare(runs):
        w.writerow([label, f"{ms:.6f}", f"{sp:.4f}"])
    return buf.getvalue()


def component_spans(trace) -> dict[int, tuple[int, float, float]]:
    """component -> (device, first start, last finish)."""
    _require(trace)
    spans = {}
    for r in trace:
        c = r["component"]
        d, a, b = spans.get(c, (r["device"], r["start"], r["finish"]))
        spans[c] = (d, min(a, r["start"]), max(b, r["finish"]))
    return spans


def component_gaps(trace, dispatch_order=None) -> list[dict]:
    """Device idle time between consecutive components on the same logical
    device: start(first command of the next component) - finish(last command of
    the previous one). In dynamic mode this is the host round trip the paper
    blames for the gaps in Fig. 12 (callback -> scheduler -> dispatch -> launch);
    in graph mode it is the event-join latency. `dispatch_order`: components in
    dispatch order (default: by start time)."""
    spans = component_spans(trace)
    order = list(dispatch_order) if dispatch_order is not None else sorted(spans, key=lambda c: spans[c][1])
    last = {}
    gaps = []
    for c in order:
        if c not in spans:
            continue
        d, a, b = spans[c]
        if d in last:
            pc, pb = last[d]
            gaps.append({"device": d, "prev": pc, "next": c, "gap": a - pb})
        last[d] = (c, b)
    return gaps


def audit_queue_order(trace) -> list[str]:
    """SPEC.md:423 trace audit: within one (component, device, queue) the commands
    start no earlier than their in-queue predecessor finished. Returns violations."""
    bad = []
    by_q = {}
    for r in sorted(trace, key=lambda r: r.get("event", 0)):
        by_q.setdefault((r["component"], r["device"], r["queue"]), []).append(r)
    for key, rs in by_q.items():
        for a, b in zip(rs, rs[1:]):
            if b["start"] + 1e-9 < a["finish"]:
                bad.append(f"{key}: {b.get('label')} starts at {b['start']} before {a.get('label')} ends at {a['finish']}")
    return bad


__all__ = ["makespan", "gantt", "compare", "compare_csv", "component_spans", "component_gaps",
           "audit_queue_order"]
