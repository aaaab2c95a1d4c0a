"""Pin the hand-built V-path fixtures (tests/vpaths.py) on the CPU checkers: a chain of
k diamonds carries exactly 2^k V-paths, and the reference's count_paths throws
overflow_error from k = 64 on -- also when the paths end at dead junctions only
(path_matrix.cpp:188-219).  The GPU side is tests/test_gpu_overflow.py."""
import os

import numpy as np
import pytest

from oracle.pyoracle import ORC_SO, REF_SO, CheckerError, Oracle64, Ref
from tests.vpaths import diamond_chain


@pytest.mark.parametrize("checker", ["ref", "oracle64"])
@pytest.mark.parametrize("k,end,overflows", [(7, "saddle", False), (63, "saddle", False), (64, "saddle", True),
                                             (63, "dead", False), (64, "dead", True),
                                             (63, "dead2", False), (64, "dead2", True)])
def test_diamond_chain_counts(checker, k, end, overflows):
    path = REF_SO if checker == "ref" else ORC_SO
    if not os.path.exists(path):
        pytest.skip(f"{path} not built")
    c = Ref() if checker == "ref" else Oracle64()
    codes, dims, src, _ = diamond_chain(k, end)
    marked, ones, twos = c.mark(codes, dims, np.array([src], c.ID))
    mn = c.minor(codes, dims, marked, ones, twos)
    if overflows:
        with pytest.raises(CheckerError) as e:
            c.count_paths(mn)
        assert e.value.kind == "overflow_error"
        return
    a, b, p = c.count_paths(mn)
    if end == "saddle":
        assert len(p) == 3 and all(int(x) == 1 << k for x in p)
    else:
        assert len(p) == 0
