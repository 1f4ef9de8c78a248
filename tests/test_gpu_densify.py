"""Densification on the device (densify.py:36-160) vs the reference's own outputs
(tests/golden/densify.npz, made by tests/golden/make_golden.py) and the oracle restatement.
fp64 throughout: 1e-12 absolute on probabilities, exact dominant materials / featureless flags.
Rows with an exact similarity tie at the k-th place are excluded from value parity (the reference
resolves those with np.argpartition; see tests/test_oracle.py::boundary_ties)."""

import numpy as np
import pytest

import paper_2511_03126_b200 as pf
import recipes
from oracle import propfield_oracle as O
from paper_2511_03126_b200 import _lib
from paper_2511_03126_b200.errors import MaterialError
from paper_2511_03126_b200.types import MaterialDictionary, MaterialEntry, SemanticPointCloud
from test_oracle import boundary_ties

pytestmark = pytest.mark.gpu


def test_dino_knn_reference_cases(cuda, golden):
    g = golden("densify")
    for name, q, s, p, k in recipes.densify_cases():
        out = pf.dino_knn_interpolate(q, s, p, k)
        keep = ~boundary_ties(q, s, k)
        np.testing.assert_allclose(out[keep], g[f"dk_{name}"][keep], rtol=0, atol=1e-12, err_msg=name)
        np.testing.assert_allclose(out.sum(axis=1), 1.0, atol=1e-9)
        # boundary-tie rows: the oracle's lower-index choice
        np.testing.assert_allclose(out, O.dino_knn_interpolate(q, s, p, k), rtol=0, atol=1e-12, err_msg=name)


def test_dino_knn_neighbour_order(cuda):
    """Neighbour indices come out in the reference's order (similarity desc, index asc)."""
    import torch

    _, q, s, p, k = [c for c in recipes.densify_cases() if c[0] == "anchors150_k5"][0]
    qd = torch.from_numpy(q).cuda()
    sd = torch.from_numpy(s).cuda()
    pd = torch.from_numpy(p).cuda()
    out = torch.empty((q.shape[0], p.shape[1]), dtype=torch.float64, device="cuda")
    nbr = torch.empty((q.shape[0], k), dtype=torch.int32, device="cuda")
    ws = torch.empty(int(_lib.load().pf_dino_knn_workspace_bytes(q.shape[0], s.shape[0], s.shape[1])),
                     dtype=torch.uint8, device="cuda")
    _lib.call("pf_dino_knn_interpolate", qd.data_ptr(), q.shape[0], sd.data_ptr(), s.shape[0], s.shape[1],
              pd.data_ptr(), p.shape[1], k, out.data_ptr(), nbr.data_ptr(), ws.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    sims = (q / np.linalg.norm(q, axis=1)[:, None]) @ (s / np.linalg.norm(s, axis=1, keepdims=True)).T
    idx = np.broadcast_to(np.arange(s.shape[0]), sims.shape)
    want = np.lexsort((idx, -sims), axis=1)[:, :k]
    got = nbr.cpu().numpy()
    # same neighbour lists except where the device's fp64 dot products round differently from BLAS
    # on a near-tie (checked through the similarity gap)
    diff = np.flatnonzero((got != want).any(axis=1))
    for i in diff:
        srt = -np.sort(-sims[i])
        assert np.min(np.abs(np.diff(srt[: k + 1]))) < 1e-13, i


def test_dino_knn_errors(cuda):
    with pytest.raises(MaterialError, match=r"\[1\]"):
        pf.dino_knn_interpolate(np.array([[1.0, 0, 0], [0, 0, 0]]), np.eye(3), np.eye(3), 1)
    with pytest.raises(ValueError):
        pf.dino_knn_interpolate(np.eye(2), np.eye(2), np.eye(2), 3)
    with pytest.raises(ValueError):
        pf.dino_knn_interpolate(np.eye(2), np.eye(2), np.eye(2), 0)


def test_dino_knn_torch_in_torch_out_and_chunks(cuda, monkeypatch):
    import torch

    from paper_2511_03126_b200 import densify

    rng = np.random.default_rng(5)
    q = rng.standard_normal((2500, 32))
    q[2100] = 0.0
    s = rng.standard_normal((70, 32))
    p = rng.dirichlet(np.ones(6), size=70)
    monkeypatch.setattr(densify, "QUERY_CHUNK", 1000)  # the missing row sits in the third chunk
    with pytest.raises(MaterialError, match=r"\[2100\]"):
        pf.dino_knn_interpolate(q, s, p, 4)
    q[2100] = 1.0
    out = pf.dino_knn_interpolate(torch.from_numpy(q).cuda(), s, p, 4)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    np.testing.assert_allclose(out.cpu().numpy(), O.dino_knn_interpolate(q, s, p, 4), rtol=0, atol=1e-12)


def test_densify_field_reference_case(cuda, golden):
    g = golden("densify")
    c = recipes.densify_field_case()
    sem = SemanticPointCloud(positions=c["positions"], features=c["features"], visible_counts=c["counts"],
                             visibility=(c["counts"] > 0)[:, None])

    class Src:
        features = c["src_features"]
        probabilities = c["src_probs"]

        def __len__(self):
            return c["src_features"].shape[0]

    entries = [MaterialEntry(name=nm, properties={"density": tuple(c["density"][i]), "hardness": tuple(c["hardness"][i])},
                             thickness_m=0.01) for i, nm in enumerate(["wood", "steel"])]
    fld = pf.densify_field(sem, Src(), MaterialDictionary(entries=entries), k=3)
    np.testing.assert_allclose(fld.probabilities, g["df_probabilities"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(fld.dominant, g["df_dominant"])
    np.testing.assert_array_equal(fld.flags["featureless"], g["df_featureless"])
    np.testing.assert_allclose(fld.properties["density"], g["df_density"], rtol=1e-12)
    np.testing.assert_allclose(fld.properties["hardness"], g["df_hardness"], rtol=1e-12)
    assert fld.material_names == ["wood", "steel"]


def test_dino_knn_pipeline_scale(cuda):
    """Pipeline-like scale: 200k fused-feature queries (D=768) against 150 anchors, k=5."""
    rng = np.random.default_rng(9)
    s = rng.standard_normal((150, 768))
    p = rng.dirichlet(np.ones(32), size=150)
    q = rng.standard_normal((200_000, 768))
    out = pf.dino_knn_interpolate(q, s, p, 5)
    rows = rng.choice(q.shape[0], 2000, replace=False)
    keep = ~boundary_ties(q[rows], s, 5)
    np.testing.assert_allclose(out[rows][keep], O.dino_knn_interpolate(q[rows], s, p, 5)[keep], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out.sum(axis=1), 1.0, atol=1e-9)


def test_nearest_grid_equals_brute_force(cuda):
    """pf_nearest_index_grid == the brute-force scan (lowest index on exact ties), including duplicated
    donors, queries outside the donors' bbox and a surface-like donor set of 300k points."""
    from paper_2511_03126_b200.densify import nearest_index

    rng = np.random.default_rng(12)
    u = rng.standard_normal((300_000, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    donors = (u * [0.4, 0.3, 0.2]).astype(np.float32).astype(np.float64)
    donors[1000:1100] = donors[0:100]  # exact ties: the lower index must win
    q = np.concatenate([donors[rng.choice(300_000, 2000)] + rng.normal(0, 1e-3, (2000, 3)),
                        rng.uniform(-1.0, 1.0, (200, 3)),  # many outside the bbox
                        donors[1000:1100]])
    g = nearest_index(q, donors, grid=True).cpu().numpy()
    b = nearest_index(q, donors, grid=False).cpu().numpy()
    np.testing.assert_array_equal(g, b)
    assert (g[-100:] == np.arange(100)).all()
