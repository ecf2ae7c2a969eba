"""GPU tau-partition (hmc_partition, NEXT-1 eqn:threshold P:200-204) against
oracle.sensitivity.partition on the same sensitivities: identical N^ and index sets (integer
work: bit-exact), both threshold rules, ties ranked by ascending index, edge cases."""
import numpy as np
import pytest

from hmcdata import ArchSpec, NetSpec, make_tiny_problem
from oracle import sensitivity as osens

from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu


def _check(S2, tau, rule):
    from paper_2507_14652_b200 import abi
    got = abi.hmc_partition(S2, tau, rule)
    ref, _ = osens.partition(S2, tau, rule)
    np.testing.assert_array_equal(got, ref.astype(np.int32))
    assert got.shape[0] == osens.n_hat(S2, tau, rule)


@pytest.mark.parametrize("P", [1, 7, 1000, 4097, 100003])
@pytest.mark.parametrize("rule", ["ge", "le"])
def test_partition_random(P, rule):
    torch_cuda()
    g = np.random.default_rng(P)
    S2 = np.exp(g.normal(-3, 2, size=P)) ** 2
    for tau in (0.5, 0.9, 0.99, 1.0):
        _check(S2, tau, rule)


@pytest.mark.parametrize("rule", ["ge", "le"])
def test_partition_ties_zeros_and_device_input(rule):
    torch = torch_cuda()
    g = np.random.default_rng(3)
    S2 = g.integers(0, 5, size=3001).astype(np.float64)   # many ties and zeros
    for tau in (0.25, 0.6, 0.95):
        _check(S2, tau, rule)
    from paper_2507_14652_b200 import abi
    dev = torch.as_tensor(S2, device="cuda")
    ref, _ = osens.partition(S2, 0.6, rule)
    np.testing.assert_array_equal(abi.hmc_partition(dev, 0.6, rule), ref.astype(np.int32))
    assert abi.hmc_partition(np.zeros(10), 0.9, rule).shape[0] == 0   # sum S^2 = 0 -> N^ = 0


def test_partition_of_gpu_sensitivities():
    """Sensitivities on the GPU, then the partition on the GPU: the same Theta_s as the oracle's
    partition of those sensitivities."""
    torch_cuda()
    from paper_2507_14652_b200 import abi
    arch = ArchSpec("mlp", (NetSpec.plain((3, 40, 30, 1)),))
    prob = make_tiny_problem(arch, n=200, seed=41)
    S2 = abi.hmc_sensitivity(prob)
    for tau in (0.9, 0.99):
        _check(S2, tau, "ge")


def test_partition_config_errors():
    torch_cuda()
    from paper_2507_14652_b200 import abi
    with pytest.raises(abi.HmcError):
        abi.hmc_partition(np.ones(5), 0.0)
    with pytest.raises(abi.HmcError):
        abi.hmc_partition(np.ones(5), 1.5)
