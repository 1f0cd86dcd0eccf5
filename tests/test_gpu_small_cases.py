"""The small cases prepared for compute-sanitizer (tools/sanitize_small.py;
the sanitizer itself is closed on the GPU pool, profiles/r2_sanitizer.txt),
run as plain parity checks against the oracle: three-/two-/one-sweep
kernels with stop replays, the cluster engine, a batched three-sweep level,
emulated row slabs with fused peer stores and the PDHG DCT kernels."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_sanitizer_small_cases():
    import sanitize_small as S

    S.cp(200, 7, resident=0, engine=6)
    S.cp(130, 5, resident=0, engine=5)
    S.cp(64, 9, resident=3)
    S.cp(40, 9, resident=0, engine=1)
    S.batch(400, 3, 8)
    S.slab(96, 3, 6)
    S.pdhg(64, 5)
