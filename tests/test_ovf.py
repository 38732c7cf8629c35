"""OVF 2.0 I/O of libmcq (B_rms maps reach Mumax3 as brmsfile.ovf, P:155;
format per SPEC's ovf-io module S:445-502).  Host-only code: runs on CPU.  Files written here by
hand (Python struct / text) pin the reader independently of the library's writer and vice versa."""
import struct

import numpy as np
import pytest


@pytest.fixture(scope="module")
def mcq():
    from _build import load_build
    load_build().build()
    import paper_2410_00966_b200 as m
    return m


HDR = """# OOMMF OVF 2.0
# Segment count: 1
# Begin: Segment
# Begin: Header
# Title: hand
# meshtype: rectangular
# meshunit: m
# valuedim: {vd}
# xnodes: {nx}
# ynodes: {ny}
# znodes: {nz}
# xstepsize: 5e-09
# ystepsize: 6e-09
# zstepsize: 7e-09
# End: Header
# Begin: Data {fmt}
"""


def _hand(path, nx, ny, nz, fmt, payload, vd=3, magic=None):
    h = HDR.format(nx=nx, ny=ny, nz=nz, fmt=fmt, vd=vd)
    if magic:
        h = h.replace("# OOMMF OVF 2.0", magic)
    with open(path, "wb") as f:
        f.write(h.encode())
        f.write(payload)
        f.write(f"\n# End: Data {fmt}\n# End: Segment\n".encode())


def test_hand_written_text_and_binary(mcq, tmp_path):
    p = tmp_path / "one.ovf"
    _hand(p, 1, 1, 1, "Text", b"0 0 1\n")
    v, g, c = mcq.mcq_ovf_read(p)
    assert g == (1, 1, 1) and c == (5e-09, 6e-09, 7e-09)
    assert v.tolist() == [[0.0, 0.0, 1.0]]
    rng = np.random.default_rng(1)
    a = rng.normal(size=(2 * 3 * 2, 3))
    p8 = tmp_path / "b8.ovf"
    _hand(p8, 2, 3, 2, "Binary 8", struct.pack("<d", 123456789012345.0) + a.astype("<f8").tobytes())
    v, g, _ = mcq.mcq_ovf_read(p8)
    assert g == (2, 3, 2) and np.array_equal(v, a.astype(np.float32))      # x fastest, as stored
    p4 = tmp_path / "b4.ovf"
    _hand(p4, 2, 3, 2, "Binary 4", struct.pack("<f", 1234567.0) + a.astype("<f4").tobytes())
    v, _, _ = mcq.mcq_ovf_read(p4)
    assert np.array_equal(v, a.astype(np.float32))


@pytest.mark.parametrize("rep", ["text", "binary4", "binary8"])
def test_round_trip_bitwise_and_deterministic(mcq, tmp_path, rep):
    rng = np.random.default_rng(7)
    a = rng.normal(size=(4 * 4 * 2, 3)).astype(np.float32) * np.float32(1e-4)
    grid, cell = (4, 4, 2), (7.8125e-9, 7.8125e-9, 2.5e-9)
    p1, p2 = tmp_path / "a.ovf", tmp_path / "b.ovf"
    mcq.mcq_ovf_write(p1, a, grid, cell, rep)
    mcq.mcq_ovf_write(p2, a, grid, cell, rep)
    assert p1.read_bytes() == p2.read_bytes()
    v, g, c = mcq.mcq_ovf_read(p1)
    assert g == grid and c == cell and np.array_equal(v, a)


def test_writer_layout_read_independently(mcq, tmp_path):
    a = np.arange(2 * 2 * 1 * 3, dtype=np.float32).reshape(-1, 3)
    p = tmp_path / "w.ovf"
    mcq.mcq_ovf_write(p, a, (2, 2, 1), (1e-9, 2e-9, 3e-9), "binary4")
    raw = p.read_bytes()
    assert raw.startswith(b"# OOMMF OVF 2.0\n") and b"\r" not in raw
    i = raw.index(b"# Begin: Data Binary 4\n") + len(b"# Begin: Data Binary 4\n")
    assert struct.unpack("<f", raw[i:i + 4])[0] == 1234567.0
    assert np.array_equal(np.frombuffer(raw[i + 4:i + 4 + a.nbytes], "<f4"), a.ravel())
    for key in (b"# xnodes: 2\n", b"# ynodes: 2\n", b"# znodes: 1\n", b"# valuedim: 3\n", b"# meshtype: rectangular\n"):
        assert key in raw


def test_errors(mcq, tmp_path):
    a = np.zeros((2, 3))
    cases = {
        "check value": ("Binary 8", struct.pack("<d", 1.0) + a.astype("<f8").tobytes(), {}),
        "truncated": ("Binary 4", struct.pack("<f", 1234567.0) + a.astype("<f4").tobytes()[:12], {}),
        "valuedim": ("Text", b"0 0 1\n0 0 1\n", {"vd": 1}),
        "OVF 2.0": ("Text", b"0 0 1\n0 0 1\n", {"magic": "# OOMMF OVF 1.0"}),
    }
    for word, (fmt, payload, kw) in cases.items():
        p = tmp_path / f"e_{word.replace(' ', '_')}.ovf"
        _hand(p, 2, 1, 1, fmt, payload, **kw)
        with pytest.raises(mcq.MCQError) as e:
            mcq.mcq_ovf_read(p)
        assert word.lower() in str(e.value).lower(), (word, str(e.value))
    p = tmp_path / "short_text.ovf"
    _hand(p, 2, 1, 1, "Text", b"0 0 1\n0 0\n")
    with pytest.raises(mcq.MCQError, match="truncated"):
        mcq.mcq_ovf_read(p)
