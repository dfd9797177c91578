"""GPU spectral diagnostics (one fused term pass per power-iteration step) vs the reference.

Golden: tests/golden/spectral.npz from the reference's spectral.estimate_spectral_radius
and verify_error_bound (tests/golden/make_golden.py).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_problem, load_golden

pytestmark = pytest.mark.gpu

SPECTRAL = {"c1": "c1", "noisy": "noisy4x60", "mixed": "mixed"}


@pytest.mark.parametrize("tag", sorted(SPECTRAL))
def test_spectral_radius_and_bound(tag):
    import paper_2204_12834_b200 as P
    from paper_2204_12834_b200 import spectral
    p, _ = golden_problem(SPECTRAL[tag])
    z = load_golden("spectral")
    lin = P.linearize(p)
    for j in range(2):
        pre = f"{tag}_l{j}_"
        s = lin.damp(float(z[pre + "lam"]))
        want = z[pre + "rho_loose"]
        est = spectral.estimate_spectral_radius(s, tol=1e-4, max_iter=20000, seed=0)
        assert est.converged == bool(want[2])
        assert abs(est.iterations - int(want[1])) <= 2
        assert abs(est.value - want[0]) <= 1e-6 * want[0]
        rep = spectral.verify_error_bound(s, [0, 1, 2, 4, 8])
        assert abs(rep.rho - float(z[pre + "rho_dense"])) <= 1e-8
        np.testing.assert_allclose(rep.measured_error, z[pre + "measured"], rtol=1e-5)
        np.testing.assert_allclose(rep.bound, z[pre + "bound"], rtol=1e-5)
        np.testing.assert_allclose([rep.u_inv_norm, rep.b_tilde_norm], z[pre + "norms"], rtol=1e-9)
        # the dense reference spectral radius bounds the power-iteration estimate
        assert est.value <= rep.rho * (1 + 1e-9)
