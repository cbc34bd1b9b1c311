"""Truncated HOSVD (paper_2211_03715_b200/tucker.py) pinned by closed forms,
the HOSVD tail-energy bound, an independent eigen-decomposition SVD oracle, the fp64
oracle's Eq. tkd2 reconstruction, and (GPU) a decomposed dense layer through the C-ABI."""
import numpy as np
import pytest

import oracle
import synth
from paper_2211_03715_b200 import tucker


def test_matricize_spec_example():
    # dims (2,2,1,1) with data [1,2,3,4], mode 1 -> [[1,3],[2,4]]
    t = np.arange(1, 5, dtype=np.float64).reshape(2, 2, 1, 1)
    assert np.array_equal(tucker.mode_n_matricize(t, 1), [[1, 3], [2, 4]])
    assert tucker.mode_n_matricize(np.zeros((64, 64, 3, 3)), 0).shape == (64, 576)
    with pytest.raises(ValueError):
        tucker.mode_n_matricize(t, 4)


def test_truncated_svd_against_eigen_oracle():
    rng = np.random.default_rng(1)
    m = rng.standard_normal((5, 7))
    u, s, v = tucker.truncated_svd(m, 2)
    assert np.allclose(u.T @ u, np.eye(2), atol=1e-12) and np.allclose(v.T @ v, np.eye(2), atol=1e-12)
    ev = np.sort(np.linalg.eigvalsh(m @ m.T))[::-1]          # independent oracle: eig of M M^T
    assert np.allclose(s, np.sqrt(ev[:2]), rtol=1e-10)
    resid = np.linalg.norm(m - u @ np.diag(s) @ v.T)
    assert abs(resid - np.sqrt(ev[2:].sum())) < 1e-9
    assert np.allclose(tucker.truncated_svd(np.eye(3), 3)[1], [1, 1, 1])
    a, b = rng.standard_normal(4), rng.standard_normal(6)
    a, b = 2 * a / np.linalg.norm(a), 3 * b / np.linalg.norm(b)
    _, s1, _ = tucker.truncated_svd(np.outer(a, b), 1)
    assert abs(s1[0] - 6.0) < 1e-12


def test_separable_kernel_rank_one_exact():
    rng = np.random.default_rng(2)
    a, b, g = rng.standard_normal(6), rng.standard_normal(5), rng.standard_normal((3, 3))
    w = np.einsum("n,c,rt->ncrt", b, a, g)
    core, u_in, u_out = tucker.tucker2_decompose(w, 1, 1)
    assert np.max(np.abs(tucker.tucker2_reconstruct(core, u_in, u_out) - w)) < 1e-12


@pytest.mark.parametrize("shape", [(4, 4, 3, 3), (16, 8, 3, 3), (12, 20, 5, 5)])
def test_full_rank_exact_and_tail_bound(shape):
    rng = np.random.default_rng(3)
    w = rng.standard_normal(shape)
    N, C = shape[:2]
    core, u_in, u_out = tucker.tucker2_decompose(w, C, N)
    assert np.max(np.abs(tucker.tucker2_reconstruct(core, u_in, u_out) - w)) < 1e-10
    for d1, d2 in [(1, 1), (C // 2, N // 2), (C, max(1, N // 3))]:
        core, u_in, u_out = tucker.tucker2_decompose(w, d1, d2)
        err = np.linalg.norm(tucker.tucker2_reconstruct(core, u_in, u_out) - w)
        assert err <= tucker.tail_energy_bound(w, d1, d2) + 1e-9
        assert np.allclose(u_in.T @ u_in, np.eye(d1), atol=1e-10)
        assert np.allclose(u_out.T @ u_out, np.eye(d2), atol=1e-10)


def test_reconstruct_agrees_with_oracle_eq_tkd2():
    rng = np.random.default_rng(4)
    w = rng.standard_normal((10, 6, 3, 3))
    core, u_in, u_out = tucker.tucker2_decompose(w, 4, 5)
    assert np.max(np.abs(tucker.tucker2_reconstruct(core, u_in, u_out)
                         - oracle.reconstruct(core, u_in, u_out))) < 1e-12


def test_decomposed_layer_equals_conv_with_projected_kernel():
    """The TKD layer built from the HOSVD factors computes conv(x, W_hat) (oracle)."""
    rng = np.random.default_rng(5)
    w = rng.standard_normal((8, 6, 3, 3))
    x = rng.standard_normal((2, 6, 9, 9))
    core, u_in, u_out = tucker.tucker2_decompose(w, 3, 4)
    y = oracle.tkd_stages(x, core, u_in, u_out, None, 2, 1)
    y_ref = oracle.conv7(x, tucker.tucker2_reconstruct(core, u_in, u_out), 2, 1)
    assert np.max(np.abs(y - y_ref)) / np.max(np.abs(y_ref)) < 1e-12


def test_rank_bounds():
    w = np.zeros((4, 3, 3, 3))
    for d1, d2 in [(0, 1), (4, 1), (1, 0), (1, 5)]:
        with pytest.raises(ValueError):
            tucker.tucker2_decompose(w, d1, d2)


@pytest.mark.gpu
def test_hosvd_factors_through_the_gpu_layer():
    """A dense 3x3 kernel, HOSVD at full rank, run as a TKD layer on the GPU (3xBF16),
    equals the dense convolution with the original kernel (oracle conv7)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2211_03715_b200 import tdc
    rng = np.random.default_rng(6)
    C, N, H = 32, 48, 12
    w = rng.standard_normal((N, C, 3, 3)) / np.sqrt(9 * C)
    core, u_in, u_out = tucker.tucker2_decompose(w, C, N)
    s = synth.LayerShape(2, C, N, H, H, C, N, 3, 1, 1)
    x = rng.uniform(-1, 1, (2, C, H, H)).astype(np.float32)
    d = {"x": x, "core": core.astype(np.float32), "u_in": u_in.astype(np.float32),
         "u_out": u_out.astype(np.float32), "bias": None}
    plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
    xd = torch.from_numpy(synth.nchw_to_nhwc(x)).cuda()
    yd = torch.empty((2, H, H, N), device="cuda")
    plan.forward(xd, yd)
    torch.cuda.synchronize()
    plan.close()
    got = synth.nhwc_to_nchw(yd.cpu().numpy()).astype(np.float64)
    ref = oracle.conv7(x, w, 1, 1)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-4
