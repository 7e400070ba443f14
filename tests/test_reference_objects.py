"""The mirror's argument handling against the REAL reference classes (CPU;
skipped where /root/reference is absent, e.g. on the GPU box): the objects
Engine.search passes to run_search (index.py:314-319) — OverlayGraph,
ProviderSource(provider, store.get), EmbeddingCache({id: vector}) — resolve
to the device inputs INTEGRATION.md §1 describes, and Engine.search with
run_search rebound to the mirror reaches the device path (DeviceError here:
no GPU in this container) instead of failing on an argument."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def engine(tmp_path_factory):
    sys.path.insert(0, str(REF))
    from slimvec.builder import BuildParams
    from slimvec.index import Engine, build_index_dir
    from slimvec.store import ItemStore
    from slimvec.vectors import ProviderConfig
    ix = tmp_path_factory.mktemp("ref") / "index"
    ItemStore.create(ix, [b"doc %d" % i for i in range(300)]).close()
    config = ProviderConfig(kind="synthetic", dim=32, seed=1, max_batch=32)
    build_index_dir(ix, BuildParams(ef_construction=24, max_degree=8, hub_percent=5.0), config)
    eng = Engine.open(ix, config)
    yield eng
    eng.close()


def test_overlay_resolves_to_base_then_to_a_frozen_snapshot(engine):
    from paper_2506_08276_b200.search import as_pruned
    ov = engine.mutable.overlay
    assert as_pruned(ov) is ov.base
    engine.add([b"new doc"])                      # inserts: the overlay overrides rows
    g = as_pruned(ov)
    assert g is not ov.base and g.n == ov.n == 301
    frozen = ov.freeze(ov.max_degree)
    for lvl in range(frozen.level_count):
        assert np.array_equal(g.level_offsets[lvl], frozen.level_offsets[lvl])
        assert np.array_equal(g.level_neighbors[lvl], frozen.level_neighbors[lvl])
    assert as_pruned(ov) is g                     # cached while the overlay is unchanged


def test_reference_sources_and_cache_resolve(engine):
    from slimvec.search import EmbeddingCache, MatrixSource, ProviderSource, SearchReport
    from paper_2506_08276_b200.search import _cache_ids, _cache_rows, _source_kind
    src = ProviderSource(engine.provider, engine.store.get)
    assert _source_kind(src) == "callback"
    rows = src.fetch([3, 5], SearchReport())
    assert rows.shape == (2, 32)
    assert _source_kind(MatrixSource(rows)) == "matrix"
    cache = EmbeddingCache({7: rows[0], 2: rows[1]})
    ids = _cache_ids(cache)
    assert list(ids) == [2, 7]
    assert np.array_equal(_cache_rows(cache, ids), np.stack([rows[1], rows[0]]))


def test_engine_search_reaches_the_device_path(engine, monkeypatch):
    import slimvec.index
    from slimvec.search import SearchParams
    from paper_2506_08276_b200.errors import DeviceError
    from paper_2506_08276_b200.search import run_search
    monkeypatch.setattr(slimvec.index, "run_search", run_search)
    with pytest.raises(DeviceError):
        engine.search(np.ones(32, np.float32), SearchParams(k=3, ef=16))


def test_reference_engine_opens_a_directory_written_here(tmp_path, monkeypatch):
    """index.build's directory layout (graph/pq/deleted/items/meta/mutations) is
    opened by the reference's own Engine.open (index.py:235-274): meta keys,
    provider hash, loaders and the item store all accept it. The GPU encoder
    registers as an external-kind provider, whose reference client requires an
    endpoint (SLIMVEC_ENDPOINT) before the caller swaps in EncoderProvider."""
    monkeypatch.setenv("SLIMVEC_ENDPOINT", "unix:/tmp/lv-encoder.sock")
    import shutil
    from conftest import GOLDEN
    from slimvec.index import Engine, read_meta as ref_read_meta
    from paper_2506_08276_b200.builder import GpuBuildParams
    from paper_2506_08276_b200.encoder import TokenStore
    from paper_2506_08276_b200.graph import load_graph, save_deleted
    from paper_2506_08276_b200.index import meta_for, read_meta, write_meta
    src = GOLDEN / "small_cos"
    g = load_graph(src / "graph.bin")
    d = tmp_path / "ix"
    d.mkdir()
    shutil.copy(src / "graph.bin", d / "graph.bin")
    shutil.copy(src / "pq.bin", d / "pq.bin")
    save_deleted(g.deleted, d / "deleted.bin")
    TokenStore(np.arange(g.n * 4, dtype=np.uint16).reshape(g.n, 4)).save(d)
    dim = int(np.load(src / "matrix.npy").shape[1])
    write_meta(d / "meta.txt", meta_for(GpuBuildParams(max_degree=g.max_degree), g.n, dim))
    (d / "mutations.log").write_bytes(b"")
    assert ref_read_meta(d / "meta.txt") == read_meta(d / "meta.txt")
    eng = Engine.open(d)
    try:
        assert eng.dim == dim and eng.mutable.overlay.n == g.n and eng.metric == "cosine"
    finally:
        eng.close()
