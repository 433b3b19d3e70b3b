"""CPU-side checks: the C-ABI library loads and exports every symbol include/skinnyqr_b200.h
declares, fails loudly without a GPU (no CPU fallback), and the host-side mirror of the reference
interface (plans, errors, slab partition) behaves like the reference."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "skinnyqr_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sqb_[a-zA-Z0-9_]+)\s*\(", text)))


def test_header_symbols_are_exported(sq):
    lib = sq.load_library()
    names = declared_symbols()
    assert len(names) >= 45
    for name in names:
        assert hasattr(lib, name), f"{name} declared in include/skinnyqr_b200.h but not exported"
    assert sorted(sq.ABI_SYMBOLS) == names


def test_no_cpu_fallback_without_gpu(sq):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sq.CudaError):
        sq.Context(0)
    with pytest.raises(sq.CudaError):
        sq.tsqr_qless(np.ones((10, 2)))


def test_product_never_imports_oracle():
    for path in (ROOT / "paper_2603_20889_b200").rglob("*"):
        if path.suffix in {".py", ".cu", ".cuh", ".h", ".hpp", ".cpp"}:
            text = path.read_text()
            assert "import oracle" not in text and "oracle/" not in text and "liboracle" not in text, path


def test_status_to_exception_mapping(sq):
    expect = {-1: sq.DimensionError, -2: sq.ArgumentError, -3: sq.BreakdownError,
              -4: sq.SingularFactorError, -5: sq.ZeroMatrixError, -6: sq.RankDeficiencyError,
              -7: sq.Error, -8: sq.CudaError, -9: sq.NcclError}
    for code, cls in expect.items():
        with pytest.raises(cls) as ei:
            sq._raise(code, 5, "test")
        if code == -3:
            assert ei.value.pivot_index == 5
        if code in (-4, -6):
            assert ei.value.diagonal_index == 5
        assert issubclass(cls, sq.Error)


def test_panel_plan_matches_reference_partition(sq, port):
    for m, k, b in [(1003, 7, 16), (10, 4, 8), (5000, 13, 48), (64, 64, 1), (1, 3, 2)]:
        plan = sq.PanelPlan(k, b)
        for blk in range(k):
            assert (plan.block_begin(m, blk), plan.block_end(m, blk)) == port.block_range(m, k, b, blk)
        covered = sum(plan.block_end(m, i) - plan.block_begin(m, i) for i in range(k))
        assert covered == m
    with pytest.raises(sq.ArgumentError):
        sq.PanelPlan(0, 4).validate()


def test_sign_normalize(sq):
    r = np.array([[-2.0, 5.0, 7.0], [0.0, 3.0, -1.0], [0.0, 0.0, -4.0]])
    out = sq.sign_normalize(r)
    assert np.array_equal(out, [[2.0, -5.0, -7.0], [0.0, 3.0, -1.0], [0.0, 0.0, 4.0]])


def test_slab_bounds(sq):
    from paper_2603_20889_b200.sharding import slab_bounds
    for m, world in [(10**9, 8), (10, 4), (3, 8), (0, 2)]:
        spans = [slab_bounds(m, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert slab_bounds(10**9, 8, 3) == (375000000, 500000000)


def test_c_abi_argument_checks_do_not_need_a_device(sq):
    lib = sq.load_library()
    assert lib.sqb_status_string(0).decode() == "ok"
    assert "Breakdown" in lib.sqb_status_string(-3).decode()
    ctx = ctypes.c_void_p()
    assert lib.sqb_create(ctypes.byref(ctx), 0) in (0, -8)
    assert lib.sqb_sync(None) == -2 and lib.sqb_destroy(None) == 0
