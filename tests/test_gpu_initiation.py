"""initiate_diffusion (integrator.py:214-265), the scalar closed-form
initiation, against the reference's own sequences (tests/golden/
initiation.npz) bit for bit, plus the reference's initiation tests
(test_integrator.py:182-265) on this path."""

import numpy as np
import pytest

from conftest import assert_bitwise, load_golden

pytestmark = pytest.mark.gpu

G = load_golden("initiation.npz")
DIR = {None: 0.0, "beta_to_alpha_s": 1.0, "alpha_s_to_beta": 2.0}
START = {"a2b": (0.9, 0.0, 0.1), "b2a": (0.0, 0.0, 1.0), "melt": (0.9, 0.0, 0.1),
         "cold": (0.9, 0.0, 0.1)}


@pytest.fixture(scope="module")
def pkg():
    import paper_2402_17580_b200 as p
    return p


@pytest.mark.parametrize("name", sorted({k.split("/")[0] for k in G.files}))
def test_sequences_match_reference(pkg, name):
    from paper_2402_17580_b200.integrator import initiate_diffusion
    t, dt, n = G[f"{name}/args"]
    st, seed = pkg.PhaseState(*START[name.split("_")[0]]), None
    rows = []
    for _ in range(int(n)):
        st, seed = initiate_diffusion(st, t, dt, seed)
        rows.append([st.x_alpha_s, st.x_alpha_m, st.x_beta, float(seed.active),
                     DIR[seed.direction], seed.tracked])
    assert_bitwise(np.array(rows), G[f"{name}/rows"], name)


def test_reference_initiation_properties(pkg):
    from paper_2402_17580_b200.integrator import analytic_beta_growth, initiate_diffusion
    from paper_2402_17580_b200.kinetics import diffusion_rate_k, x_alpha_eq
    out, seed = initiate_diffusion(pkg.PhaseState(0.9, 0.0, 0.1), 1200.0, 1e-4, None)
    assert seed.direction == "alpha_s_to_beta" and seed.active
    assert 0.0 < seed.tracked < 1e-30 and out.x_beta == pytest.approx(0.1, abs=1e-15)
    _, expected = analytic_beta_growth(1200.0, 1e-4, 1)
    assert (out.x_beta - 0.1) == pytest.approx(expected[0] - 0.1, rel=1e-8)
    _, k_b = diffusion_rate_k(1200.0)
    delta = 0.9 - x_alpha_eq(1200.0)
    assert seed.tracked == pytest.approx(delta / (1.0 + (11.0 / (delta * k_b * 1e-4)) ** 11.0),
                                         rel=1e-8)
    # hand-off: tracked * dt crosses the initiation threshold
    st, sd = pkg.PhaseState(0.9, 0.0, 0.1), None
    for _ in range(10000):
        st, sd = initiate_diffusion(st, 1200.0, 0.01, sd)
        if not sd.active:
            break
    assert not sd.active and sd.tracked * 0.01 > 1e-15
    # the kernels' seed pass and the scalar op agree (test_integrator.py:256-265)
    kseed = pkg.SeedingState()
    kout = pkg.step_explicit(pkg.PhaseState(0.9, 0.0, 0.1), 1200.0, 1200.0, 1e-4, seeding=kseed)
    assert kseed.active == seed.active
    assert kseed.tracked == pytest.approx(seed.tracked, rel=1e-13)
    assert kout.x_beta == pytest.approx(out.x_beta, abs=1e-16)
