"""Device numerics the bit-exactness argument rests on.

* ``div_rcp(a, b, rcp_nr(b))`` — one refined reciprocal shared by several
  quotients — equals ``__ddiv_rn`` bit for bit on every operand class the
  kernels feed it (and on a wide log-uniform class as a stress test);
* K2's filtered ``rint((f*x)/z + c)`` equals the correctly rounded
  expression, including quotients within 1e-9 of a rounding boundary;
* K0's ``(float)mm / 1000`` via reciprocal + FMA correction equals the IEEE
  quotient for all 65,536 u16 inputs (core.py:264 uses true division).
"""

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,n", [(0, 1 << 28), (1, 1 << 28), (2, 1 << 28), (3, 1 << 27),
                                    (4, 1 << 26), (5, 1 << 16)])
def test_shared_reciprocal_division_matches_ddiv_rn(cuda, mode, n):
    import torch

    from paper_2007_00558_b200 import _native

    ctx = _native.context()
    bad = torch.zeros(1, dtype=torch.int64, device=cuda)
    ctx.call("fvv_selftest_division", n, 20071007 + mode, mode, bad.data_ptr())
    assert int(bad.item()) == 0
