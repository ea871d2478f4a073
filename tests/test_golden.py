"""Product vs golden fixtures captured from the reference's own L0-L2 code
(tests/golden/reference_l0_l2.json, made by tests/golden/make_golden.py).
Runs anywhere — no /root/reference needed."""
import json
import pathlib

import pytest

from paper_2009_07482_b200 import _native

FIX = pathlib.Path(__file__).with_name("golden") / "reference_l0_l2.json"
FIXTURES = json.loads(FIX.read_text()) if FIX.exists() else []


def _q(req):
    import ctypes
    L = _native.lib()
    p = L.hs_query(json.dumps(req).encode())
    try:
        return json.loads(ctypes.string_at(p).decode())
    finally:
        L.hs_free_string(p)


def test_fixture_file_present():
    assert len(FIXTURES) > 200


@pytest.mark.parametrize("i", range(len(FIXTURES)))
def test_matches_reference_fixture(i):
    req, ref = FIXTURES[i]["request"], FIXTURES[i]["response"]
    ours = _q({**req, "json_style": "cudnn-fe"} if req["op"] == "parse" else req)
    if not ref["ok"]:
        assert not ours["ok"] and ours["errc"] == ref["errc"] and ours.get("exit") == ref.get("exit"), (ours, ref)
    else:
        assert ours == ref
