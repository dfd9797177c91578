"""Host-only covisibility clustering (libpoba poba_cluster_cameras) vs the reference's cluster_cameras."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_problem, load_golden

POST = {"c1": "c1", "mixed": "mixed", "c2": "c2"}


@pytest.mark.parametrize("tag", sorted(POST))
@pytest.mark.parametrize("size", [1, 5, 16, 1000])
def test_cluster_cameras_matches_reference(tag, size):
    from paper_2204_12834_b200 import clustering
    p, _ = golden_problem(POST[tag])
    z = load_golden("post")
    part = clustering.cluster_cameras(p, size)
    pre = f"{tag}_s{size}_"
    assert np.array_equal(part.assignment, z[pre + "assignment"])
    assert [part.n_clusters, part.cut_observations] == z[pre + "meta"].tolist()
    assert np.array_equal(part.sizes, z[pre + "sizes"])
    assert part.sizes.max() <= size


def test_cluster_size_must_be_positive():
    from paper_2204_12834_b200 import clustering
    p, _ = golden_problem("c1")
    with pytest.raises(ValueError, match="max_cluster_size must be at least 1"):
        clustering.cluster_cameras(p, 0)
