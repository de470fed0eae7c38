"""Artifact formats: .zgla tensors, ledger.csv, timeline.json are byte-compatible
with the reference writers (glasp/tensorio.py, glasp/reports.py)."""

import struct

import numpy as np
import pytest

from paper_2507_01004_b200 import reports, tensorio
from paper_2507_01004_b200.cluster import Event, LedgerRow, VirtualTimeline, VolumeLedger
from paper_2507_01004_b200.errors import TensorFormatError


def test_zgla_layout_by_hand(tmp_path):
    a = np.arange(6, dtype=np.float64).reshape(2, 3) * 0.5
    p = tmp_path / "a.zgla"
    tensorio.write_tensor(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"ZGLA" and struct.unpack("<3I", raw[4:16]) == (2, 2, 3) and len(raw) == 16 + 48
    assert np.array_equal(tensorio.read_tensor(p), a)


def test_zgla_torch_bf16_widened(tmp_path):
    torch = pytest.importorskip("torch")
    t = torch.tensor([[1.5, -2.25]], dtype=torch.bfloat16)
    p = tmp_path / "t.zgla"
    tensorio.write_tensor(p, t)
    assert np.array_equal(tensorio.read_tensor(p), np.array([[1.5, -2.25]]))


@pytest.mark.parametrize("raw", [b"", b"XXXX\x01\x00\x00\x00", b"ZGLA\x02\x00\x00\x00\x01\x00",
                                 b"ZGLA\x01\x00\x00\x00\x02\x00\x00\x00" + b"\x00" * 8])
def test_zgla_malformed(tmp_path, raw):
    p = tmp_path / "bad.zgla"
    p.write_bytes(raw)
    with pytest.raises(TensorFormatError):
        tensorio.read_tensor(p)


def _ledger():
    return VolumeLedger(2, (LedgerRow(1, "all_scan", 0, 16384), LedgerRow(0, "all_scan", 16384, 0)))


def test_ledger_and_timeline_render():
    csv = reports.ledger_csv(_ledger())
    assert csv == "rank,primitive,sent_elements,received_elements\n0,all_scan,16384,0\n1,all_scan,0,16384\n"
    tl = VirtualTimeline((Event(0, "local_scan", 0.0, 1.5e-05),))
    js = reports.timeline_json(tl)
    assert '"label": "local_scan"' in js and js.endswith("\n")


@pytest.mark.reference
def test_byte_identical_to_reference_writers(tmp_path):
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from glasp import reports as ref_reports
    from glasp import tensorio as ref_io
    from glasp.cluster import VolumeLedger as RefLedger

    a = np.random.default_rng(0).standard_normal((2, 3, 4))
    ours, theirs = tmp_path / "o.zgla", tmp_path / "t.zgla"
    tensorio.write_tensor(ours, a)
    ref_io.write_tensor(theirs, a)
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(ref_io.read_tensor(ours), a)
    rows = [{"rank": 0, "primitive": "all_scan", "sent_elements": 3, "received_elements": 0, "x": 0.1}]
    cols = ("rank", "primitive", "sent_elements", "received_elements", "x")
    assert reports.render_csv(rows, cols) == ref_reports.render_csv(rows, cols)
    assert reports.render_json(rows, cols) == ref_reports.render_json(rows, cols)
    assert RefLedger is not None
