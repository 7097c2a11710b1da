"""Device field generator (csrc/grf.cu) against its CPU restatement
(oracle/grf_oracle.py): Philox4x32-10 known answers, the DCT matrix, and the
sampled fields of every config kind at reduced and at full size."""

import numpy as np
import pytest
import scipy.fft as sfft

from oracle import grf_oracle as go
from paper_2401_09516_b200 import problems as P

SEED = P.BASE_SEED


# Philox4x32-10 known-answer vectors (Random123 kat_vectors: counter, key -> output)
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_oracle_philox_known_answers(ctr, key, out):
    r = go.philox4x32_10(*[np.array([c]) for c in ctr], *key)
    assert tuple(int(v[0]) for v in r) == out


def test_oracle_normals_statistics():
    z = go.normals(200001, SEED, 3, 5, 0)
    assert z.shape == (200001,)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    u = go.uniforms(100001, SEED, 2, 0, 1)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    # streams / systems / configs are independent draws
    assert not np.array_equal(go.normals(8, SEED, 3, 5, 0), go.normals(8, SEED, 3, 6, 0))
    assert not np.array_equal(go.normals(8, SEED, 3, 5, 0), go.normals(8, SEED, 3, 5, 1))


@pytest.mark.parametrize("n", [2, 7, 64, 128])
def test_dct_matrix_is_scipy_idct(n):
    T = P.dct_matrix(n)
    v = np.random.default_rng(n).standard_normal(n)
    np.testing.assert_allclose(T @ v, sfft.idct(v, type=2, norm="ortho"), rtol=0, atol=1e-13)
    np.testing.assert_allclose(T @ T.T, np.eye(n), atol=1e-13)


def test_oracle_field_laws():
    f = go.system_params("darcy_binary", 2, 32, 3.0, 1.0, SEED, 0, 4)
    assert set(np.unique(f["a"])) <= {3.0, 12.0}
    assert 0.2 < np.mean(f["a"] == 12.0) < 0.8
    assert abs(np.mean(f["g"] ** 2) - 1.0) < 0.6  # unit mean pointwise variance (one sample)
    h = go.system_params("helmholtz", 2, 32, 3.0, 1.0, SEED, 2, 4)
    assert 10.0 <= h["k0"] < 20.0 and np.all((h["center"] >= 0.2) & (h["center"] < 0.8))
    assert h["params"].shape == (32 * 32 + 1,)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    return torch


@pytest.mark.gpu
def test_device_philox_matches_oracle():
    torch = _cuda()
    from paper_2401_09516_b200 import _lib

    L = _lib.load()
    for count, cid, idx, stream in ((1, 0, 0, 0), (1001, 3, 77, 0), (65536, 1, 0, 7)):
        z = torch.empty(count, dtype=torch.float64, device="cuda")
        assert L.skr_philox_normals(count, SEED, cid, idx, stream, 1.0, z.data_ptr(), None) == 0
        ref = go.normals(count, SEED, cid, idx, stream)
        np.testing.assert_allclose(z.cpu().numpy(), ref, rtol=1e-14, atol=1e-15)
    u = torch.empty(5, dtype=torch.float64, device="cuda")
    assert L.skr_philox_uniforms(5, SEED, 2, 9, 1, u.data_ptr(), None) == 0
    # uniforms are exact (integer -> double conversions and one power-of-two scale)
    assert np.array_equal(u.cpu().numpy(), go.uniforms(5, SEED, 2, 9, 1))


def _check_field(spec, idx):
    torch = _cuda()
    f = P.system_params_device(spec, idx)
    torch.cuda.synchronize()
    ref = go.system_params(spec.kind, spec.dim, spec.n, spec.tau, spec.scale, SEED, spec.cid, idx)
    g_ref = ref["g"]
    scale = np.abs(g_ref).max()
    if spec.kind == "helmholtz":
        assert f["k0"] == ref["k0"]
        np.testing.assert_array_equal(f["center"], ref["center"])
        g = f["g"].cpu().numpy()
        np.testing.assert_allclose(g, g_ref, rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(f["kfield"].cpu().numpy(), ref["kfield"], rtol=1e-13)
        p = f["params"].cpu().numpy()
        assert p[0] == ref["k0"]
        np.testing.assert_allclose(p[1:], g_ref.ravel(), rtol=0, atol=1e-12 * scale)
        return
    a = f["a"].cpu().numpy()
    if spec.kind == "darcy_binary":
        # the thresholded field is exact wherever g is not within rounding of 0
        safe = np.abs(g_ref) > 1e-10 * scale
        assert safe.mean() > 0.999
        np.testing.assert_array_equal(a[safe], ref["a"][safe])
    else:
        np.testing.assert_allclose(a, ref["a"], rtol=1e-12)
    np.testing.assert_array_equal(f["params"].cpu().numpy(), a.ravel())


@pytest.mark.gpu
@pytest.mark.parametrize("cid,n,idx", [(0, 64, 0), (0, 64, 255), (1, 64, 3), (2, 48, 5),
                                       (3, 24, 1), (4, 96, 2)])
def test_device_field_matches_oracle_reduced(cid, n, idx):
    _check_field(P.CONFIGS[cid].reduced(n=n), idx)


@pytest.mark.gpu
@pytest.mark.parametrize("cid,idx", [(0, 7), (1, 11), (2, 1), (3, 0), (4, 3)])
def test_device_field_matches_oracle_full_size(cid, idx):
    """BASELINE sizes: 64^2, 256^2, 256^2, 128^3 (2.1 M cells), 1024^2."""
    _check_field(P.CONFIGS[cid], idx)


@pytest.mark.gpu
def test_device_generated_chain_matches_host_assembly():
    """params_device -> device sort -> device assembly: the systems equal the
    host assembly of the oracle's fields (bit for bit), and the chain solves."""
    torch = _cuda()
    import paper_2401_09516_b200 as skr

    spec = P.CONFIGS[0].reduced(n=24, n_systems=6)
    flat, extra = P.params_device(spec)
    order = skr.greedy_sort_device(flat)
    ref_flat = np.stack([go.system_params(spec.kind, 2, 24, spec.tau, 1.0, SEED, 0, i)["params"]
                         for i in range(6)])
    assert np.array_equal(flat.cpu().numpy(), ref_flat)
    from oracle import skr_oracle as orc

    assert order == orc.greedy_order(ref_flat)
    systems = []
    for i in range(6):
        fields = P.fields_from_params_device(spec, flat[i], extra[i])
        dA, b, _ = P.assemble_device(spec, i, fields, jacobi=False)
        rp, ci, v, bh, _ = P.assemble(spec, i, {"a": ref_flat[i].reshape(24, 24),
                                                 "params": ref_flat[i]})
        assert np.array_equal(dA.values.cpu().numpy(), v)
        assert np.array_equal(b.cpu().numpy(), bh)
        systems.append((dA, b))
    cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=1e-8, max_iter=2000)
    res = skr.solve_sequence(systems, order, cfg, "none", keep_x="none")
    assert all(res.converged)
