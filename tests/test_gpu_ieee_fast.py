"""The branch-free FP64 fast paths of csrc/ieee_fast.cuh return the IEEE round-to-nearest
result bit for bit whenever their range check passes (DESIGN "Kernels": the pointwise
stage runs on them and falls back to the IEEE operators otherwise, so dt stays
bit-exact).  ~2e8 seeded operands per (op, distribution) on the device."""
from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2104_11404_b200 import hydro  # noqa: E402


@pytest.mark.parametrize("op", [0, 1, 2], ids=["div", "rcp", "sqrt"])
@pytest.mark.parametrize("dist", [0, 1], ids=["typical", "rawbits"])
def test_fast_paths_bit_exact(op, dist):
    bad, slow, tot = hydro.selftest_ieee_fast(0x2104_11404 + 7 * op + dist, 1 << 27, op, dist)
    torch.cuda.synchronize()
    assert tot == 1 << 27
    assert bad == 0, f"{bad} fast-path results differ from IEEE"
    if dist == 0:
        # typical operands must almost always stay on the fast path
        assert slow <= tot // 1000, (slow, tot)
