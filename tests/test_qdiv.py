"""Host check of the kernels' division-free block-index decomposition
(`qdiv` in csrc/he_internal.cuh): for 0 <= x < 2^20 and 1 <= d < 2^20,
floor((x + 1/2) * r) == x // d whenever r is within 2 ulp of 1/d in float32
(the hardware reciprocal `rcp.approx.ftz.f32` is within 1 ulp).  Float32
arithmetic emulated with numpy; every x below 2^20 for each divisor."""
import numpy as np
import pytest

DIVISORS = list(range(1, 65)) + [100, 127, 255, 256, 1000, 1536, 3072, 4095,
                                 65535, 99991, (1 << 20) - 1]


@pytest.mark.parametrize("d", DIVISORS)
def test_qdiv_float_reciprocal_exact(d):
    x = np.arange(1 << 20, dtype=np.int64)
    xf = x.astype(np.float32) + np.float32(0.5)          # exact: x < 2^23
    want = x // d
    r0 = np.float32(1.0) / np.float32(d)
    rs = [r0]
    for direction in (np.float32(0), np.float32(np.inf)):
        r = r0
        for _ in range(2):                                 # 1 and 2 ulp away
            r = np.nextafter(r, direction, dtype=np.float32)
            rs.append(r)
    for r in rs:
        got = np.floor(xf * np.float32(r)).astype(np.int64)   # float32 product
        assert np.array_equal(got, want), (d, float(r))
