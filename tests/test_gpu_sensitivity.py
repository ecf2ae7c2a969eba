"""GPU sensitivities (hmc_sensitivity, eqn:sensitivities P:193-197) against the fp64 oracle's
definition (one reverse pass per datum), and the tau-partition (eqn:threshold) built from them."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_problem, make_tiny_problem
from oracle import sensitivity as osens

from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

# fp32 sums of squares over the data (3xTF32 or FMA): relative error ~1e-6 per entry; the
# north_star tolerance (1e-5) on the norm and on every entry that is not ~1e3 times below the max
REL2 = 1e-5      # ||S2_gpu - S2_ref|| / ||S2_ref||
RELI = 1e-5      # per entry, relative to the entry, for entries >= 1e-3 max


def _data(prob):
    if prob.arch.kind == "mlp":
        return {"x": prob.x, "y": prob.y}
    return {"u": prob.u, "q": prob.q, "v": prob.v}


def _check(prob):
    torch_cuda()
    from paper_2507_14652_b200 import abi
    got = abi.hmc_sensitivity(prob)
    ref = osens.sensitivities(prob.arch, prob.frozen.astype(np.float64), prob.sigma_vi.astype(np.float64),
                              _data(prob))
    assert got.shape == ref.shape and np.all(got >= 0)
    r2 = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert r2 <= REL2, r2
    big = ref >= 1e-3 * ref.max()
    ri = np.max(np.abs(got[big] - ref[big]) / ref[big])
    assert ri <= RELI, ri
    # the partition the paper's Algorithm 2 builds from them: bit-exact (same N^, same index set)
    # whenever the oracle's own margins at the cut exceed the measured error - the gap between the
    # last selected and the first unselected score, and the distance of the cumulative fractions
    # c_{N^-1}, c_{N^} from tau; otherwise (a cut inside the rounding band) N^ within 1
    err = np.abs(got - ref)
    n_exact = 0
    for tau in (0.5, 0.9, 0.99):
        n_r = osens.n_hat(ref, tau)
        order = np.lexsort((np.arange(ref.size), -ref))
        srt = ref[order]
        csum = np.cumsum(srt) / srt.sum()
        e_tot = err.sum() / srt.sum()
        gap_ok = n_r >= srt.size or (srt[n_r - 1] - srt[n_r]) > err[order[n_r - 1]] + err[order[n_r]]
        c_ok = abs(csum[n_r - 1] - tau) > 2 * e_tot and (n_r < 2 or abs(csum[n_r - 2] - tau) > 2 * e_tot)
        n_g = osens.n_hat(got, tau)
        if gap_ok and c_ok:
            n_exact += 1
            assert n_g == n_r, (tau, n_g, n_r)
            np.testing.assert_array_equal(osens.partition(got, tau)[0], osens.partition(ref, tau)[0])
        else:
            assert abs(n_g - n_r) <= 1, (tau, n_g, n_r)
    return got, ref, n_exact


CASES = {
    "mlp_ragged_simt": (ArchSpec("mlp", (NetSpec.plain((3, 50, 30, 1)),)), dict(n=77)),
    "mlp_tc": (ArchSpec("mlp", (NetSpec.plain((2, 64, 96, 1)),)), dict(n=300)),
    "mlp_sin": (ArchSpec("mlp", (NetSpec((1, 8, 1), ("sin", "identity"), (True, True)),)), dict(n=40)),
    "deeponet_tc": (ArchSpec("deeponet", (NetSpec.plain((5, 64, 64, 32)),
                                          NetSpec.plain((2, 64, 32), last="tanh")), has_b0=True),
                    dict(n_c=24, n_x=40)),
    "deeponet_ragged": (ArchSpec("deeponet", (NetSpec.plain((7, 30, 10)), NetSpec.plain((3, 20, 10), last="tanh")),
                                 has_b0=False), dict(n_c=13, n_x=17)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_sensitivity_matches_oracle(name):
    arch, kw = CASES[name]
    prob = make_tiny_problem(arch, seed=21, **kw)
    _check(prob)


def test_sensitivity_cfg2_full_size():
    """cfg2 (MLP 1-64x4-1, N = 1024) at full size; its cuts at tau = 0.5 and 0.9 lie 1e-3 / 8e-4
    (score gap) and 1.3e-3 / 1.8e-5 (cumulative fraction) away from any tie, far outside the
    ~1e-6 rounding band, so those partitions must be bit-exact (tau = 0.99's cut is 7e-7 from
    c_{N^-1} and may legitimately move by one)."""
    _, _, n_exact = _check(make_problem("cfg2", n_chains=1))
    assert n_exact >= 2


def test_sensitivity_cfg4_shape_deeponet():
    """cfg4's DeepONet widths (branch 100-128-128-128-100, trunk 1-128-128-100, b0) on 24 x 30
    pairs (the oracle's per-pair reverse passes bound the size)."""
    full = make_problem("cfg4", n_chains=1)
    full.u = np.ascontiguousarray(full.u[:24])
    full.q = np.ascontiguousarray(full.q[:30])
    full.v = np.ascontiguousarray(full.v[:24, :30])
    got, ref, _ = _check(full)
    b0 = full.frozen.shape[0] - 1
    assert got[b0] == pytest.approx(float(full.sigma_vi[b0]) ** 2, rel=1e-6)   # dF/db0 = 1


def test_sensitivity_scale_and_zero_sigma():
    torch_cuda()
    from paper_2507_14652_b200 import abi
    arch, kw = CASES["mlp_tc"]
    prob = make_tiny_problem(arch, seed=5, **kw)
    s1 = abi.hmc_sensitivity(prob)
    sig = prob.sigma_vi.astype(np.float32) * 2.0
    sig[7] = 0.0
    s2 = abi.hmc_sensitivity(prob, sigma_vi=sig)
    mask = np.arange(s1.size) != 7
    np.testing.assert_allclose(s2[mask], 4.0 * s1[mask], rtol=1e-12)
    assert s2[7] == 0.0
