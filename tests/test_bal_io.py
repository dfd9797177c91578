"""Native BAL ingest (libpoba poba_bal_parse) against the reference's own parse_bal.

tests/golden/bal.npz holds a corpus of BAL texts and what the reference's
bal_io.parse_bal made of each (arrays, pruning counts, or the exact error).
Host-only: runs without a GPU.
"""
from __future__ import annotations

import io

import numpy as np
import pytest

from conftest import load_golden

Z = load_golden("bal")
CASES = sorted(k[:-5] for k in Z if k.endswith("_text") and k != "rig_text")
KEYS = ("camera_params", "points", "cam_indices", "pt_indices", "pixels")


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype.kind == b.dtype.kind and np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["text", "bytes", "path"])
def test_corpus_matches_reference(name, mode, tmp_path):
    from paper_2204_12834_b200 import bal_io
    text = bytes(Z[f"{name}_text"]).decode()
    if mode == "text":
        src = io.StringIO(text)
    elif mode == "bytes":
        src = io.BytesIO(text.encode())
    else:
        if "\r" in text:
            pytest.skip("text-mode files translate line endings (line numbers may differ from a stream)")
        src = tmp_path / f"{name}.bal"
        src.write_text(text)
    if bool(Z[f"{name}_ok"]):
        p = bal_io.parse_bal(src)
        for k in KEYS:
            assert _eq(getattr(p, k), Z[f"{name}_{k}"]), (name, k)
        assert [p.n_pruned_cameras, p.n_pruned_points] == Z[f"{name}_pruned"].tolist()
    else:
        kind, msg = str(Z[f"{name}_error"]).split(": ", 1)
        assert kind == "BalParseError"
        with pytest.raises(bal_io.BalParseError) as e:
            bal_io.parse_bal(src)
        assert str(e.value) == msg
        assert isinstance(e.value, ValueError)


def test_round_trip_file_bit_exact(tmp_path):
    """serialize_bal output of the reference (repr floats) parses to identical arrays."""
    from paper_2204_12834_b200 import bal_io
    path = tmp_path / "rig.bal"
    path.write_bytes(bytes(Z["rig_text"]))
    p = bal_io.parse_bal(str(path))
    assert p.name == "rig"
    for k in KEYS:
        assert _eq(getattr(p, k), Z[f"rig_{k}"]), k


def test_bytes_stream_must_be_ascii():
    from paper_2204_12834_b200 import bal_io
    with pytest.raises(UnicodeDecodeError):
        bal_io.parse_bal(io.BytesIO("1 1 1\n0 0 1 2\n\xe9\n".encode("latin-1")))


def test_large_synthetic_round_trip(tmp_path):
    """A C3-scale file (880k observations) parses and matches the generator's arrays."""
    from paper_2204_12834_b200 import bal_io, configs
    p = configs.make_config("c3", 0.25)
    lines = [f"{p.n_cameras} {p.n_points} {p.n_observations}"]
    lines += [f"{c} {q} {x!r} {y!r}" for c, q, (x, y) in zip(p.cam_indices.tolist(), p.pt_indices.tolist(),
                                                          p.pixels.tolist())]
    lines += [repr(v) for v in p.camera_params.ravel().tolist()] + [repr(v) for v in p.points.ravel().tolist()]
    path = tmp_path / "c3.bal"
    path.write_text("\n".join(lines) + "\n")
    q = bal_io.parse_bal(path)
    for k in KEYS:
        assert _eq(getattr(q, k), getattr(p, k)), k
