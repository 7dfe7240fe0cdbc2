"""The reference's vectorised model API (kinetics.py:144-269) and the
polynomial helpers (fastmath.py:261-303), bit for bit against
tests/golden/kinetics_api.npz; the exponentials run on the device."""

import numpy as np
import pytest

from conftest import assert_bitwise, load_golden

pytestmark = pytest.mark.gpu

G = load_golden("kinetics_api.npz")


@pytest.fixture(scope="module")
def pkg():
    import paper_2402_17580_b200 as p
    return p


def test_model_functions_bitwise(pkg):
    from paper_2402_17580_b200 import kinetics as k
    t, xs, xm = G["t"], G["xs"], G["xm"]
    assert_bitwise(k.liquid_fraction(t), G["liquid_fraction"], "g")
    assert_bitwise(k.solid_fraction(t), G["solid_fraction"], "xsol")
    assert_bitwise(k.x_alpha_eq(t), G["x_alpha_eq"], "xaeq")
    assert_bitwise(k.x_alpha_m_eq(t, xs), G["x_alpha_m_eq"], "xmeq")
    kas, kb = k.diffusion_rate_k(t)
    assert_bitwise(kas, G["k_as"], "k_as")
    assert_bitwise(kb, G["k_b"], "k_b")
    r = k.compute_rates((xs, xm), t)
    assert_bitwise(r.d_x_alpha_s, G["ds"], "ds")
    assert_bitwise(r.d_x_alpha_m, G["dm"], "dm")
    st = k.apply_corrections((xs, xm), t)
    assert_bitwise(st.x_alpha_s, G["cxs"], "cxs")
    assert_bitwise(st.x_alpha_m, G["cxm"], "cxm")
    assert_bitwise(st.x_beta, G["cxb"], "cxb")


def test_scalar_forms(pkg):
    for (a, b, tt), ref in zip(G["scalar_in"], G["scalar_out"]):
        r = pkg.compute_rates(pkg.PhaseState(a, b, 0.0), tt)
        c = pkg.apply_corrections(pkg.PhaseState(a, b, 0.0), tt)
        got = [r.d_x_alpha_s, r.d_x_alpha_m, c.x_alpha_s, c.x_alpha_m, c.x_beta,
               pkg.x_alpha_eq(tt), pkg.liquid_fraction(tt)]
        assert all(isinstance(v, float) for v in got)
        assert_bitwise(np.array(got), ref, f"scalar {a},{b},{tt}")
