"""R31 level schedule of eps (opts.eps_decay) through the C ABI against the oracle."""
import pytest

from synth import uniform_points
import paper_2506_16759_b200 as g
from gpu_helpers import oracle_build, compare_builds

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("decay", [0.8, 1.5])
def test_eps_decay_parity(decay):
    X = uniform_points(4096, 3, 2)
    Ho, _ = oracle_build(X, "exp", 0.2, 64, 1e-6, eps_decay=decay)
    Hg = g.build(g.Tree(X, 64), ("exp", 0.2), 1e-6, eps_decay=decay)
    assert Hg.samples == Ho.samples
    certified, compared = compare_builds(Hg, Ho)
    assert certified <= max(2, compared // 50)
