"""Host polynomial helpers (fastmath.py:261-303) and the coefficient tables
against the reference (tests/golden/kinetics_api.npz, fastmath.npz)."""

import numpy as np

from conftest import assert_bitwise, load_golden
from paper_2402_17580_b200 import batch
from paper_2402_17580_b200.fastmath import (EXP_CORRECTION, LN_CORRECTION, estrin_eval,
                                            horner_eval)

G = load_golden("kinetics_api.npz")


def test_estrin_horner_bitwise():
    y = G["y"]
    assert_bitwise(estrin_eval(EXP_CORRECTION, y), G["estrin_exp"], "estrin exp")
    assert_bitwise(estrin_eval(LN_CORRECTION, y), G["estrin_ln"], "estrin ln")
    assert_bitwise(estrin_eval((1.0, -0.5, 0.25, 0.125, -1.5), y), G["estrin_odd"], "odd")
    assert_bitwise(horner_eval(LN_CORRECTION, y), G["horner_ln"], "horner ln")
    assert isinstance(estrin_eval(EXP_CORRECTION, 0.5), float)


def test_blend_and_dispatch():
    assert batch.branch_dispatch([True, True]) == "all"
    assert batch.branch_dispatch([False, False]) == "none"
    assert batch.branch_dispatch([True, False]) == "some"
    assert np.array_equal(batch.blend(np.array([True, False]), 1.0, 2.0), [1.0, 2.0])


def test_device_tables_match_python_tables():
    import re
    from pathlib import Path
    src = (Path(batch.__file__).parent / "csrc" / "ti64_fastmath.cuh").read_text()
    ea = {int(k): float(v) for k, v in re.findall(r"\bEA(\d) = ([-+0-9.eE]+)", src)}
    lb = {int(k): float(v) for k, v in re.findall(r"\bLB(\d+) = ([-+0-9.eE]+)", src)}
    assert tuple(ea[i] for i in range(8)) == EXP_CORRECTION.coefficients
    assert tuple(lb[i] for i in range(12)) == LN_CORRECTION.coefficients
