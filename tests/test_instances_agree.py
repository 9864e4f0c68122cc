"""One instance definition: the host problems
(instances.sqeuclid_problem / rect_problem, used by the e2e bench leg and the
reference fixtures) and the device-generated ones (DeviceProblem.sqeuclid_grid
/ rect_l1, used by the device-resident bench leg and the tests) are the same
instance bit for bit: f, g, cost_fro_norm and marginal_norm on the host (CPU
test), the cost matrix itself on the device (GPU test).

The marginals are the reference's marginal_from_image: the raw image weights
normalised ONCE (instance.py:153-158)."""


import numpy as np
import pytest

CASES = [("c1", dict(r=32)), ("c2", dict(r=64)), ("c3", dict(r=128)), ("c4", dict(rect=True))]


def _host(inst, case):
    return inst.rect_problem(0) if case.get("rect") else inst.sqeuclid_problem(case["r"], 0)


def _device_vectors(inst, case):
    """The f, g, norms DeviceProblem.generated uploads (device.py), computed on the host."""
    if case.get("rect"):
        m, n = 8192, 32768
        f, g = inst.sparse_marginals(m, 0), inst.sparse_marginals(n, 1)
        fro = inst.rect_l1_fro_norm()
    else:
        f, g = inst.whitenoise_marginals(case["r"], 0)
        fro = inst.sqeuclid_fro_norm(case["r"])
    return f, g, fro, float(np.linalg.norm(f) + np.linalg.norm(g))


@pytest.mark.parametrize("name,case", CASES)
def test_host_and_device_instances_agree(name, case):
    from paper_2407_19689_b200 import instances as inst
    prob = _host(inst, case)
    f, g, fro, marg = _device_vectors(inst, case)
    assert np.array_equal(prob.f, f) and np.array_equal(prob.g, g)
    assert prob.cost_fro_norm == fro
    assert prob.marginal_norm == marg
    # normalised once: the reference's Marginal(raw) (w / w.sum()) bit for bit
    if not case.get("rect"):
        src, dst = inst.whitenoise_images(case["r"], 0)
        assert np.array_equal(f, src.ravel() / float(src.ravel().sum()))
        assert np.array_equal(g, dst.ravel() / float(dst.ravel().sum()))


@pytest.mark.parametrize("r", [8, 16, 32, 64])
def test_exact_norm_equals_reference_norm(r):
    """Up to r = 64 the integer sum of squares is exact in fp64, so the exact norm the
    device problem uses equals the reference's np.linalg.norm(C)."""
    from paper_2407_19689_b200 import instances as inst
    assert float(np.linalg.norm(inst.sqeuclid_grid_cost(r))) == inst.sqeuclid_fro_norm(r)


@pytest.mark.gpu
@pytest.mark.parametrize("name,case", [c for c in CASES if c[0] != "c3"])
def test_device_cost_equals_host_cost(name, case):
    import torch

    import paper_2407_19689_b200 as pd
    from paper_2407_19689_b200 import instances as inst
    prob = _host(inst, case)
    dp = pd.DeviceProblem.rect_l1(0) if case.get("rect") else pd.DeviceProblem.sqeuclid_grid(case["r"], 0)
    assert np.array_equal(dp.f_t.cpu().numpy(), prob.f) and np.array_equal(dp.g_t.cpu().numpy(), prob.g)
    assert dp.cost_fro_norm == prob.cost_fro_norm and dp.marginal_norm == prob.marginal_norm
    C = torch.from_numpy(np.asarray(prob.C)).to(dp.C_t.device)
    assert torch.equal(dp.C_t[:, :prob.n], C)
