"""score_views / rank_views on the device (view_select.py:51-124) vs the reference's
outputs on 150 anchors of the `mini` workload (tests/golden/views.npz): ranked view indices exact,
scores / depths / pixels within 1e-12."""

import numpy as np
import pytest

from paper_2511_03126_b200 import view_select, workloads

pytestmark = pytest.mark.gpu


class Src:
    def __init__(self, positions, normals):
        self.positions, self.normals, self.flags = positions, normals, {}

    def __len__(self):
        return self.positions.shape[0]


def test_rank_views_matches_reference(cuda, golden):
    g = golden("views")
    wl = workloads.generate("mini")
    src = Src(wl.points.astype(np.float64)[g["indices"]], g["normals"])
    st, sa, z, px = view_select.score_views(src, wl.views(f32_maps=True), g["visibility"])
    np.testing.assert_allclose(st, g["s_total"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(sa, g["s_angle"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(z, g["z"])
    np.testing.assert_array_equal(px, g["pixels"])
    ranks = view_select.rank_views(src, wl.views(f32_maps=True), g["visibility"], 3)
    got = np.full((len(ranks), 3), -1, np.int32)
    for i, r in enumerate(ranks):
        for q, e in enumerate(r):
            got[i, q] = e.view_index
            assert e.point_index == i and e.s_dist == pytest.approx(1.0 / (1.0 + e.z), rel=1e-15)
    np.testing.assert_array_equal(got, g["ranked"])
    np.testing.assert_array_equal(src.flags["zero_visible"], g["zero_visible"])
    with pytest.raises(ValueError):
        view_select.rank_views(src, wl.views(f32_maps=True), g["visibility"], 0)
    src.normals = None
    with pytest.raises(ValueError):
        view_select.score_views(src, wl.views(f32_maps=True), g["visibility"])
