"""CPU-side checks of the C-ABI boundary: the library builds, loads and exports
every entry point declared in include/leann_b200.h (no compute without a GPU)."""
from __future__ import annotations

import re

import pytest

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "leann_b200.h").read_text()
    return sorted(set(re.findall(r"\b(lv_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for required in ("lv_index_create", "lv_search_batch", "lv_adc_tables", "lv_adc_score",
                     "lv_distance_many", "lv_encoder_create", "lv_encode", "lv_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import __graft_entry__ as ge
    ge.build()
    from paper_2506_08276_b200 import _lib
    lib = _lib.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.lv_version() == 1


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.errors import DeviceError
    g = lv.load_graph(ROOT / "tests" / "golden" / "small_cos" / "graph.bin")
    m, c = lv.load_pq(ROOT / "tests" / "golden" / "small_cos" / "pq.bin")
    with pytest.raises(DeviceError):
        lv.DeviceIndex(g, m, c)


def test_search_params_validation():
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.errors import InvalidArgumentError
    for kw in (dict(k=0), dict(k=5, ef=3), dict(rerank_percent=0.0), dict(batch_size=0),
               dict(mode="dfs"), dict(cache_percent=101.0)):
        with pytest.raises(InvalidArgumentError):
            lv.SearchParams(**kw)


def test_formats_round_trip(tmp_path):
    import numpy as np
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.errors import FormatError
    d = ROOT / "tests" / "golden" / "small_cos"
    g = lv.load_graph(d / "graph.bin")
    lv.save_graph(g, tmp_path / "g.bin")
    assert (tmp_path / "g.bin").read_bytes() == (d / "graph.bin").read_bytes()
    m, c = lv.load_pq(d / "pq.bin")
    lv.save_pq(m, c, tmp_path / "p.bin")
    assert (tmp_path / "p.bin").read_bytes() == (d / "pq.bin").read_bytes()
    data = (d / "graph.bin").read_bytes()
    for cut in (3, 10, len(data) - 2):
        (tmp_path / "t.bin").write_bytes(data[:cut])
        with pytest.raises(FormatError):
            lv.load_graph(tmp_path / "t.bin")
    (tmp_path / "t.bin").write_bytes(data + b"zz")
    with pytest.raises(FormatError) as err:
        lv.load_graph(tmp_path / "t.bin")
    assert "trailing" in str(err.value)
    bad = bytearray(data)
    bad[:4] = b"NOPE"
    (tmp_path / "t.bin").write_bytes(bytes(bad))
    with pytest.raises(FormatError) as err:
        lv.load_graph(tmp_path / "t.bin")
    assert err.value.section == "graph.magic"
    dl = np.zeros(g.n, bool)
    dl[::7] = True
    lv.save_deleted(dl, tmp_path / "d.bin")
    assert np.array_equal(lv.load_deleted(tmp_path / "d.bin", g.n), dl)


def test_validate_catches_violations():
    import numpy as np
    import paper_2506_08276_b200 as lv
    from paper_2506_08276_b200.errors import FormatError

    def mk(rows, max_degree=4):
        off = np.zeros(len(rows) + 1, np.uint64)
        flat = []
        for v, r in enumerate(rows):
            flat.extend(r)
            off[v + 1] = len(flat)
        return lv.PrunedGraph(n=len(rows), max_degree=max_degree, entry_point=0,
                              levels=np.zeros(len(rows), np.uint16), level_offsets=[off],
                              level_neighbors=[np.asarray(flat, np.uint32)])
    lv.validate(mk([[1], [0]]))
    for rows, md in (([[0], []], 4), ([[1, 1], [], []], 4), ([[1, 2, 3], [], [], []], 2),
                     ([[7], []], 4)):
        with pytest.raises(FormatError):
            lv.validate(mk(rows, md))


def test_tune_ef_matches_reference_semantics():
    """evaluation.py:132-161 ported cases (reference tests/test_evaluation.py:92-104)."""
    from paper_2506_08276_b200.evaluation import tune_ef

    def evaluate(ef):
        return min(1.0, ef / 50.0)

    r = tune_ef(evaluate, k=3, n=100, target_recall=0.0)
    assert r.ef == 3 and r.feasible
    r = tune_ef(evaluate, k=3, n=100, target_recall=0.9)
    assert r.feasible and r.ef == 45
    assert evaluate(r.ef) >= 0.9 > evaluate(r.ef - 1)
    bad = tune_ef(lambda ef: 0.5, k=3, n=100, target_recall=0.9)
    assert not bad.feasible and bad.ef == 100
    # a dip below the target just under the endpoint raises the non-monotone warning
    flip = tune_ef(lambda ef: 1.0 if ef in (40, 41) or ef >= 45 else 0.0, 3, 100, 0.9)
    assert flip.feasible


def test_recall_at_k_reference_semantics():
    from paper_2506_08276_b200.evaluation import mean_recall, recall_at_k
    from paper_2506_08276_b200.errors import InvalidArgumentError
    assert recall_at_k([1, 2, 3], [3, 4, 5]) == 1 / 3
    assert mean_recall([[1, 2], [5, 6]], [[1, 2], [6, 7]]) == 0.75
    with pytest.raises(InvalidArgumentError):
        recall_at_k([1], [])


def test_index_create_rejects_rows_beyond_max_degree_and_bad_ids():
    """lv_index_create validates every CSR row before touching the device
    (frontier scratch is sized from max_degree; bitmaps are indexed by id)."""
    import ctypes as C
    import numpy as np
    from paper_2506_08276_b200 import _lib

    def create(offsets, nbrs, max_degree):
        offs = np.asarray(offsets, dtype=np.uint64)
        nb = np.asarray(nbrs, dtype=np.uint32)
        d = _lib.IndexDesc()
        d.n, d.dim, d.metric, d.max_degree, d.level_count = len(offs) - 1, 4, 2, max_degree, 1
        d.entry_point = 0
        op = (C.c_void_p * 1)(offs.ctypes.data)
        npp = (C.c_void_p * 1)(nb.ctypes.data)
        nnz = (C.c_uint64 * 1)(nb.shape[0])
        d.level_offsets = C.cast(op, C.POINTER(C.c_void_p))
        d.level_neighbors = C.cast(npp, C.POINTER(C.c_void_p))
        d.level_nnz = C.cast(nnz, C.POINTER(C.c_uint64))
        h = C.c_void_p()
        rc = _lib.lib().lv_index_create(C.byref(d), 0, C.byref(h))
        return rc, _lib.lib().lv_last_error().decode()

    rc, msg = create([0, 3, 3, 3], [1, 2, 1], max_degree=2)     # row 0 has 3 > M = 2
    assert rc == 3 and "exceeds M" in msg
    rc, msg = create([0, 1, 2, 2], [1, 7], max_degree=2)        # neighbour id 7 >= n = 3
    assert rc == 3 and "out of range" in msg
    rc, msg = create([0, 2, 1, 2], [1, 2], max_degree=2)        # offsets not monotone
    assert rc == 3
