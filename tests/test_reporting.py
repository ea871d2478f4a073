"""Reporting on synthetic traces: the SPEC examples for
makespan / gantt / compare, plus component gaps and the queue-order audit."""
import xml.etree.ElementTree as ET

import pytest

from paper_2009_07482_b200 import reporting as R
from paper_2009_07482_b200._native import HetsimError


def ev(i, start, finish, kind="ndrange", label=None, device=0, queue=0, component=0, channel=-1):
    return {"event": i, "kind": kind, "label": label or f"e{i + 1}", "kernel": i, "component": component,
            "device": device, "queue": queue, "channel": channel, "start": start, "finish": finish}


def test_makespan_examples():
    with pytest.raises(HetsimError) as e:
        R.makespan([])
    assert e.value.errc == "EmptyTrace" and e.value.exit_code == 2
    assert R.makespan([ev(0, 0, 14)]) == 14
    assert R.makespan([ev(0, 3, 5), ev(1, 4, 9)]) == 6


def test_gantt_text_serial_and_lanes():
    serial = [ev(0, 0, 2, "write", "w1"), ev(1, 2, 5, label="e1"), ev(2, 5, 6, "read", "r1")]
    txt = R.gantt(serial, "text", quantum=1.0)
    rows = txt.strip().splitlines()
    assert len(rows) == 1
    bar = rows[0].split("|")[1]
    assert bar == "w1e1=r"  # three non-overlapping bars in one lane
    overlapping = [ev(0, 0, 4, label="e1", queue=0), ev(1, 1, 3, label="e2", queue=1)]
    rows = R.gantt(overlapping, "text").strip().splitlines()
    assert len(rows) == 2 and rows[0].startswith("d0.q0") and rows[1].startswith("d0.q1")
    with pytest.raises(HetsimError):
        R.gantt([], "text")


def test_gantt_svg_is_well_formed():
    svg = R.gantt([ev(0, 0, 2, "write", "w1"), ev(1, 1, 3, label="e1 <k>", queue=1)], "svg")
    root = ET.fromstring(svg)
    assert root.tag.endswith("svg")
    assert len([c for c in root if c.tag.endswith("rect")]) == 2


def test_compare_examples():
    t105, t95 = [ev(0, 0, 105)], [ev(0, 0, 95)]
    assert R.compare([("a", t105), ("b", t105)]) == [("a", 105, 1.0), ("b", 105, 1.0)]
    assert R.compare([("coarse", t105), ("fine", t95)])[1][2] == 1.1053
    assert R.compare([("only", t95)]) == [("only", 95, 1.0)]
    csv = R.compare_csv([("coarse", t105), ("fine", t95)]).splitlines()
    assert csv[0] == "label,makespan_ms,speedup" and csv[2].endswith(",1.1053")


def test_component_gaps_and_audit():
    tr = [ev(0, 0, 2, component=0), ev(1, 2, 3, component=0), ev(2, 3.5, 5, component=1),
          ev(3, 0, 9, component=2, device=1), ev(4, 9.25, 10, component=3, device=1)]
    gaps = R.component_gaps(tr)
    assert [(g["prev"], g["next"], g["gap"]) for g in gaps] == [(0, 1, 0.5), (2, 3, 0.25)]
    assert R.audit_queue_order(tr) == []
    assert R.audit_queue_order([ev(0, 0, 2), ev(1, 1, 3)])  # overlap inside one queue is flagged
