"""CPU-side checks of the boundary: the library loads, exports every symbol include/mcq.h
declares, and the binding's constants match the header.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mcq.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"MCQ_API\s+[^;(]*?\b(mcq_\w+)\s*\(", txt)))


def _defines():
    txt = open(HEADER).read()
    return {k: int(v.rstrip("u"), 0) for k, v in re.findall(r"#define\s+(MCQ_\w+)\s+\(?(-?\w+)\)?", txt)
            if re.fullmatch(r"-?\d+u?", v)}


@pytest.fixture(scope="module")
def built():
    from _build import load_build
    b = load_build()
    b.build()
    return b.LIB


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("mcq_create", "mcq_set_brms", "mcq_set_cavity", "mcq_relax", "mcq_run", "mcq_get_m",
              "mcq_get_cavity", "mcq_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(built)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header_and_constants(built):
    import paper_2410_00966_b200 as mcq
    from paper_2410_00966_b200 import _lib
    assert sorted(_lib.EXPORTED) == _declared()
    for n in _declared():
        assert callable(getattr(mcq, n))
    d = _defines()
    assert d["MCQ_TERM_ALL"] == mcq.TERM_ALL == 127 and d["MCQ_TERM_DMI"] == mcq.TERM_DMI == 64
    assert (d["MCQ_TERM_ZEEMAN"], d["MCQ_TERM_EXCHANGE"], d["MCQ_TERM_ANIS"], d["MCQ_TERM_DEMAG"],
            d["MCQ_TERM_CAVITY"], d["MCQ_TERM_EXCITATION"]) == (1, 2, 4, 8, 16, 32)
    from oracle import sim as S
    assert (S.ZEEMAN, S.EXCHANGE, S.ANIS, S.DEMAG, S.CAVITY, S.EXCITATION, S.DMI) == (1, 2, 4, 8, 16, 32, 64)
    assert S.ALL == 127
    assert d["MCQ_NKCLASS"] == mcq.NKCLASS
    assert d["MCQ_TRACE_COLS"] == len(mcq.TRACE_COLS) == 8
    assert (d["MCQ_OK"], d["MCQ_EINVAL"], d["MCQ_ESTATE"]) == (0, -1, -2)


def test_create_without_gpu_fails_cleanly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2410_00966_b200 as mcq
    with pytest.raises(mcq.MCQError):
        mcq.mcq_create((8, 8, 1), (5e-9,) * 3, 1.4e5, 3.7e-12, 0.01)


def test_invalid_arguments_rejected_before_device_use(built):
    import paper_2410_00966_b200 as mcq
    for grid, cell, Ms in [((1, 8, 1), (1e-9,) * 3, 1e5), ((8, 8, 0), (1e-9,) * 3, 1e5),
                           ((8, 8, 1), (0.0, 1e-9, 1e-9), 1e5), ((8, 8, 1), (1e-9,) * 3, -1.0),
                           ((1024, 8, 1), (1e-9,) * 3, 1e5)]:
        with pytest.raises(mcq.MCQError) as e:
            mcq.mcq_create(grid, cell, Ms, 1e-11, 0.01)
        assert e.value.code == -1


def test_no_cpu_fallback_in_product_package():
    """The product package never imports the oracle (parity would be void otherwise)."""
    pkg = os.path.join(ROOT, "paper_2410_00966_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
