"""IVHG graph cache (reference knng.py:286-332) — reader/writer parity with
files the reference wrote (tests/golden/make_knn_golden.py), zero-copy
neighbour mapping, the reference's error behaviour; and (GPU) an embedding
from a cache-mapped graph equals one from the in-memory graph."""

import os

import numpy as np
import pytest

from paper_2303_05455_b200 import knng
from paper_2303_05455_b200.embed import KnnGraph
from paper_2303_05455_b200.errors import MalformedInputError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_reads_reference_cache():
    g = knng.cache_read(os.path.join(GOLD, "ref_cache_cosine.ivhg"))
    assert g.metric == "cosine" and g.neighbors.shape == (300, 4) and g.neighbors.dtype == np.int32
    raw = open(os.path.join(GOLD, "ref_cache_cosine.ivhg"), "rb").read()
    nb = np.frombuffer(raw[24:24 + 300 * 4 * 4], dtype="<u4").reshape(300, 4)
    dist = np.frombuffer(raw[24 + 300 * 16:], dtype="<f4").reshape(300, 4)
    np.testing.assert_array_equal(g.neighbors, nb)
    np.testing.assert_array_equal(g.distances, dist.astype(np.float64))
    g2 = knng.cache_read(os.path.join(GOLD, "ref_cache_nodist.ivhg"))
    assert g2.distances is None
    np.testing.assert_array_equal(g2.neighbors, g.neighbors)


def test_writer_is_byte_identical(tmp_path):
    for name in ("ref_cache_cosine.ivhg", "ref_cache_nodist.ivhg"):
        g = knng.cache_read(os.path.join(GOLD, name))
        out = tmp_path / name
        knng.cache_write(g, str(out))
        assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read()


def test_neighbours_are_mapped_not_copied(tmp_path):
    g = KnnGraph(np.arange(40, dtype=np.int32).reshape(10, 4) % 10)
    p = tmp_path / "g.ivhg"
    knng.cache_write(g, str(p))
    h = knng.cache_read(str(p))
    assert not h.neighbors.flags.owndata  # a view of the file mapping
    np.testing.assert_array_equal(h.neighbors, g.neighbors)


def test_errors(tmp_path):
    p = tmp_path / "bad.ivhg"
    p.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(MalformedInputError, match="not a graph cache"):
        knng.cache_read(str(p))
    raw = open(os.path.join(GOLD, "ref_cache_cosine.ivhg"), "rb").read()
    p.write_bytes(raw[:4] + np.asarray([2], "<u4").tobytes() + raw[8:])
    with pytest.raises(MalformedInputError, match="unsupported cache version"):
        knng.cache_read(str(p))
    p.write_bytes(raw[:-8])
    with pytest.raises(MalformedInputError, match="truncated"):
        knng.cache_read(str(p))
    with pytest.raises(MalformedInputError, match="cannot read"):
        knng.cache_read(str(tmp_path / "missing.ivhg"))


@pytest.mark.gpu
def test_embedding_from_cache_equals_in_memory(tmp_path):
    from paper_2303_05455_b200 import EmbeddingConfig, run_embedding, synth

    nb = synth.planted_graph(20000, 3, seed=4)
    p = tmp_path / "planted.ivhg"
    knng.cache_write(KnnGraph(nb), str(p))
    cfg = EmbeddingConfig(nn=3, rn=1, c=0.1, iterations=50, seed=2)
    a = run_embedding(graph=KnnGraph(nb), config=cfg)
    b = run_embedding(graph=knng.cache_read(str(p)), config=cfg)
    np.testing.assert_array_equal(a.embedding.points, b.embedding.points)
    assert a.trace.stress == b.trace.stress
