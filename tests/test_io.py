"""CPU: Γ file formats (byte-identical to the reference's serialize_gamma,
harness.py:183-250) and per-range checkpoints."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1503_08809_b200 import (GammaFormatError, GammaMatrix, deserialize_gamma,
                                   load_checkpoint, merge_checkpoints, save_checkpoint,
                                   serialize_gamma)

META = {"engine": "modal3d", "l_min": 2, "l_max": 16, "integrator": "trap",
        "tables": "t", "grid": "g", "mapping": "m"}


def desk_gamma(g_desk):
    return GammaMatrix(g_desk["desk_gamma"], dict(META))


@pytest.mark.parametrize("fmt,name", [("csv", "desk_gamma.csv"), ("bin", "desk_gamma.bin")])
def test_bytes_identical_to_reference(tmp_path, g_desk, fmt, name):
    out = tmp_path / name
    serialize_gamma(desk_gamma(g_desk), out, fmt)
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()


@pytest.mark.parametrize("fmt,name", [("csv", "desk_gamma.csv"), ("bin", "desk_gamma.bin")])
def test_read_reference_files(g_desk, fmt, name):
    g = deserialize_gamma(os.path.join(GOLDEN, name), fmt)
    assert np.array_equal(g.values, g_desk["desk_gamma"])
    if fmt == "csv":
        assert g.meta["engine"] == "modal3d" and g.meta["l_max"] == 16


def test_format_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("# nope\n1,2\n")
    with pytest.raises(GammaFormatError):
        deserialize_gamma(bad, "csv")
    bad.write_text("# modalgamma v1 engine=x nmax=2 lmin=2 lmax=3 integrator=trap\n1,2\n")
    with pytest.raises(GammaFormatError):
        deserialize_gamma(bad, "csv")
    badb = tmp_path / "bad.bin"
    badb.write_bytes(b"MGAM" + (1).to_bytes(4, "little") + (2).to_bytes(4, "little")
                     + (2).to_bytes(4, "little") + b"\0" * 8)
    with pytest.raises(GammaFormatError):
        deserialize_gamma(badb, "bin")
    with pytest.raises(ValueError):
        serialize_gamma(GammaMatrix(np.eye(2)), tmp_path / "x", "hdf5")


def test_checkpoints_merge_in_order(tmp_path):
    rng = np.random.default_rng(1)
    parts = [GammaMatrix(rng.standard_normal((5, 5)), dict(META)) for _ in range(3)]
    paths = []
    for i, g in enumerate(parts):
        p = tmp_path / f"part{i}.mgam"
        save_checkpoint(g, p, begin=i * 10, end=(i + 1) * 10)
        paths.append(p)
    g1, side = load_checkpoint(paths[1])
    assert side["range"] == [10, 20] and np.array_equal(g1.values, parts[1].values)
    merged = merge_checkpoints(paths)
    want = parts[0].values.copy()
    want += parts[1].values
    want += parts[2].values
    assert np.array_equal(merged.values, want) and merged.meta["workers_merged"] == 3
    other = GammaMatrix(np.zeros((5, 5)), dict(META, tables="other"))
    save_checkpoint(other, tmp_path / "bad.mgam")
    with pytest.raises(ValueError):
        merge_checkpoints([paths[0], tmp_path / "bad.mgam"])


def test_checkpoint_spans_are_validated(tmp_path):
    rng = np.random.default_rng(2)
    g = [GammaMatrix(rng.standard_normal((4, 4)), dict(META)) for _ in range(3)]
    paths = []
    for i, (b, e) in enumerate(((20, 35), (0, 20), (35, 50))):    # saved out of order
        p = tmp_path / f"c{i}.mgam"
        save_checkpoint(g[i], p, begin=b, end=e)
        paths.append(p)
    merged = merge_checkpoints(paths, expect=(0, 50))
    want = g[1].values.copy()
    want += g[0].values
    want += g[2].values                                              # summed in span order
    assert np.array_equal(merged.values, want)
    with pytest.raises(ValueError, match="uncovered"):
        merge_checkpoints(paths[:2], expect=(0, 50))                 # hole [35, 50)
    dup = tmp_path / "dup.mgam"
    save_checkpoint(g[0], dup, begin=30, end=40)
    with pytest.raises(ValueError, match="overlap"):
        merge_checkpoints(paths + [dup])
    slab = tmp_path / "slab.mgam"
    save_checkpoint(g[0], slab, l2_begin=2, l2_end=10)
    with pytest.raises(ValueError, match="mix"):
        merge_checkpoints([paths[0], slab])
    assert np.array_equal(merge_checkpoints([slab], expect=(2, 10)).values, g[0].values)
