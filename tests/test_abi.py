"""The C-ABI library loads and exports every symbol include/pipeoptim.h
declares; host-only entry points behave like the reference; the product path
has no CPU fallback. CPU only (no kernel launches)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "pipeoptim.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(po_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2312_00839_b200 import _lib
    from paper_2312_00839_b200.build import build_library

    build_library()
    return _lib.load()


def test_header_declares_expected_entry_points():
    from paper_2312_00839_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.po_abi_version() == 1


def test_so_is_sm100a_cubin():
    from paper_2312_00839_b200.build import LIB_PATH

    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_difference_through_abi(lib):
    from paper_2312_00839_b200.optim import version_difference

    assert version_difference(4, 0) == 3 and version_difference(4, 3) == 0 and version_difference(1, 0) == 0
    assert [version_difference(8, r) for r in range(8)] == [7, 6, 5, 4, 3, 2, 1, 0]
    for bad in ((0, 0), (4, 4), (4, -1)):
        with pytest.raises(ValueError):
            version_difference(*bad)
    out = ctypes.c_int64(-1)
    assert lib.po_version_difference(3, 3, ctypes.byref(out)) == -22
    assert lib.po_strerror(-22) == b"invalid argument"
    assert lib.po_strerror(0) == b"ok"


def test_optimizer_config_validation():
    from paper_2312_00839_b200.optim import OptimizerConfig

    for bad in (dict(kind="rmsprop"), dict(kind="sgdm", momentum=1.0), dict(kind="adam", beta2=-0.1),
                dict(kind="adam", eps=0.0), dict(kind="sgdm", dampening=1.5)):
        with pytest.raises(ValueError):
            OptimizerConfig(**bad)
    c = OptimizerConfig("adamw")
    hp = c.hparams()
    assert (hp.kind, hp.beta2, hp.decoupled_decay, hp.weight_decay) == (2, 0.999, 1e-2, 5e-4)


def test_no_cpu_fallback_without_cuda(lib):
    """On a box without a GPU the product path raises instead of computing."""
    import torch

    from paper_2312_00839_b200 import _lib
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    st = OptimizerState(OptimizerConfig("adam"), ["w"])
    with pytest.raises((_lib.LibraryMissing, RuntimeError, AssertionError)):
        st.step([torch.ones(2, 2)], [torch.ones(2, 2)], 0.1)


def test_missing_library_fails_loudly(tmp_path):
    from paper_2312_00839_b200 import _lib

    with pytest.raises(_lib.LibraryMissing):
        _lib.load(tmp_path / "libpipeoptim.so")


def test_flat_layout_alignment():
    from paper_2312_00839_b200.optim import FlatLayout

    lay = FlatLayout(["a", "b", "c"], [(3, 5), (1, 5), (7,)])
    assert lay.offsets == [0, 64, 128] and lay.numel == 192
    assert lay.locate(3) == "a" and lay.locate(66) == "b" and lay.locate(20) == "<padding>"
    import torch

    buf = torch.arange(lay.numel, dtype=torch.float32)
    views = lay.views(buf)
    assert views[1].shape == (1, 5) and float(views[1][0, 0]) == 64.0


@pytest.mark.parametrize("n,dp", [(0, 2), (10, 4), (512, 8), (70_080, 3), (1_000_003, 8), (64, 1)])
def test_dp_shard_ranges_tile_the_stage(lib, n, dp):
    """po_dp_shard_range (host-side, no GPU): contiguous shards covering
    [0, n), each starting on a 64-element (256 B) boundary."""
    spans = []
    for r in range(dp):
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        assert lib.po_dp_shard_range(n, dp, r, ctypes.byref(lo), ctypes.byref(hi)) == 0
        spans.append((lo.value, hi.value))
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(lo % 64 == 0 or lo == n for lo, _ in spans)
    lo = ctypes.c_int64()
    assert lib.po_dp_shard_range(n, dp, dp, ctypes.byref(lo), ctypes.byref(lo)) != 0
    assert lib.po_dp_shard_range(n, 9, 0, ctypes.byref(lo), ctypes.byref(lo)) != 0
