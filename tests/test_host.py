"""CPU tier: the C-ABI library and the host side of the drop-in, no GPU needed.

* libgraphlb_b200.so loads and exports exactly the functions
  include/graphlb_b200.h declares, and the ctypes table binds them all;
* the C-ABI rejects bad arguments with the documented status codes before it
  touches a device (glb_last_error carries the message);
* host-side semantics of the drop-in package follow the reference:
  generators (bit-identical arrays, pinned digests), CsrGraph validation and
  from_edges stability (csr.py:42-118), KernelConfig / resolve_threads
  (engine.py:39-70), RelaxOp, DistArray, MetricsRecord statistics
  (engine.py:142-174), verify (oracles.py:58-82), the COO budget rule
  (csr.py:155-170) and run_strategy's tag / source validation
  (strategies/__init__.py:17-41, common.py:68-70).
"""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1711_00231_b200 as pkg
from paper_1711_00231_b200 import _lib
from tests import graph_specs as gs

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "graphlb_b200.h"


def header_functions() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(glb_\w+)\s*\(", text, flags=re.M))


def test_library_exports_every_declared_function():
    names = header_functions()
    assert len(names) >= 25, names
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding covers exactly the declared surface
    assert set(_lib.SIGNATURES) == names
    _lib.lib()  # binds every signature


def test_c_abi_rejects_bad_arguments_without_a_device():
    L = _lib.lib()
    out = ctypes.c_void_p()
    row = np.array([0, 1], dtype=np.int64)
    col = np.array([0], dtype=np.int64)
    # NULL out pointer
    assert L.glb_graph_create(_lib.ptr64(row), _lib.ptr64(col), None, 1, 1, 0, None) == _lib.GLB_EINVAL
    assert b"NULL" in L.glb_last_error()
    # negative sizes
    assert L.glb_graph_create(_lib.ptr64(row), _lib.ptr64(col), None, -1, 1, 0,
                              ctypes.byref(out)) == _lib.GLB_EINVAL
    # glb_run on a NULL graph
    p, st = _lib.RunParams(), _lib.RunStats()
    assert L.glb_run(None, ctypes.byref(p), None, ctypes.byref(st), None, 0) == _lib.GLB_EINVAL
    # primitives validate before allocating
    v = np.array([1, 2], dtype=np.int64)
    assert L.glb_inclusive_scan(_lib.ptr64(v), -1, _lib.ptr64(v), 0) == _lib.GLB_EINVAL
    assert L.glb_find_offsets(_lib.ptr64(v), 2, 0, 4, _lib.ptr64(v), _lib.ptr64(v), 0) == _lib.GLB_EINVAL
    assert L.glb_measure_gather(None, None) == _lib.GLB_EINVAL
    nb, fb = ctypes.c_int64(), ctypes.c_int64()
    assert L.glb_validate(None, 0, 0, _lib.ptr64(v), ctypes.byref(nb), ctypes.byref(fb)) == _lib.GLB_EINVAL
    n = ctypes.c_int(-1)
    assert L.glb_device_count(ctypes.byref(n)) == _lib.GLB_OK and n.value >= 0
    assert L.glb_version().decode()


def test_status_codes_map_to_reference_exceptions(monkeypatch):
    monkeypatch.setattr(_lib, "lib", lambda: type("L", (), {"glb_last_error": staticmethod(lambda: b"m")})())
    for code, exc in ((_lib.GLB_EINVAL, ValueError), (_lib.GLB_ERANGE, IndexError),
                      (_lib.GLB_EOVERFLOW, OverflowError), (_lib.GLB_ENOMEM, MemoryError),
                      (_lib.GLB_ECUDA, RuntimeError), (_lib.GLB_ENODEV, RuntimeError)):
        with pytest.raises(exc):
            _lib.check(code, "x")
    _lib.check(_lib.GLB_OK)


def test_host_generators_match_reference_digests(golden):
    d = golden["generators"]["digests"]
    for gid, spec in gs.CORPUS.items():
        if gid in d:
            assert gs.digest(gs.build(pkg, spec)) == d[gid], gid


def test_csr_validation_and_stable_grouping():
    with pytest.raises(ValueError):
        pkg.CsrGraph(2, 1, [0, 1], [0])          # row length
    with pytest.raises(ValueError):
        pkg.CsrGraph(2, 1, [0, 2, 1], [0])       # end != num_edges
    with pytest.raises(ValueError):
        pkg.CsrGraph(2, 2, [0, 2, 1 + 1], [0, 5])  # col out of range
    with pytest.raises(ValueError):
        pkg.CsrGraph(1, 1, [0, 1], [0], [-1])    # negative weight
    g = pkg.CsrGraph.from_edges(3, [2, 0, 2, 0], [1, 2, 0, 1], [7, 8, 9, 10])
    assert g.row_offsets.tolist() == [0, 2, 2, 4]
    assert g.col_indices.tolist() == [2, 1, 1, 0]  # input order kept within a row
    assert g.weights.tolist() == [8, 10, 7, 9]
    assert not g.row_offsets.flags.writeable
    assert g.outdegrees().tolist() == [2, 0, 2]


def test_coo_budget_rule_is_checked_on_the_host():
    g = pkg.CsrGraph(2, 2, [0, 2, 2], [1, 0], [3, 4])
    assert pkg.graph.coo_cells_required(2, True) == 6
    with pytest.raises(pkg.CooCapacityError) as ei:
        pkg.csr_to_coo(g, max_cells=5)
    assert isinstance(ei.value, MemoryError)
    assert (ei.value.required_cells, ei.value.available_cells) == (6, 5)
    assert pkg.DEFAULT_COO_BUDGET_CELLS == 1_000_000_000


def test_kernel_config_and_resolve_threads():
    with pytest.raises(ValueError):
        pkg.KernelConfig(virtual_threads=0)
    with pytest.raises(ValueError):
        pkg.KernelConfig(block_size=0)
    with pytest.raises(ValueError):
        pkg.KernelConfig(loop="bogus")
    with pytest.raises(ValueError):
        pkg.KernelConfig(dist_bits=16)
    for bits in (0, 24, 32, 64):
        assert pkg.KernelConfig(dist_bits=bits).dist_bits == bits
    cfg = pkg.KernelConfig()
    # engine.py:63-70: min(2^14, ceil(items / block) * block), at least one block
    assert pkg.resolve_threads(cfg, 0) == 1024
    assert pkg.resolve_threads(cfg, 1025) == 2048
    assert pkg.resolve_threads(cfg, 10**9) == 1 << 14
    assert pkg.resolve_threads(pkg.KernelConfig(virtual_threads=7), 10**6) == 7


def test_relax_op_dist_array_and_records():
    with pytest.raises(ValueError):
        pkg.RelaxOp("dfs")
    assert pkg.RelaxOp("bfs").candidate(3, 100) == 4
    assert pkg.RelaxOp("sssp").candidate(3, 100) == 103
    with pytest.raises(IndexError):
        pkg.DistArray(3, source=3)
    d = pkg.DistArray(3, source=1)
    assert d.values == [pkg.INF, 0, pkg.INF] and len(d) == 3 and d[1] == 0
    assert d == [pkg.INF, 0, pkg.INF]
    work = [3, 0, 5, 8]
    listed = pkg.MetricsRecord(0, "BS", 4, work, 10, 2, 0.001)
    summed = pkg.MetricsRecord(0, "BS", 4, None, 10, 2, 0.001, n_threads=4, total_work=sum(work),
                               max_work=max(work), work_sumsq=float(sum(w * w for w in work)))
    for r in (listed, summed):
        assert r.threads == 4 and r.work_total() == 16 and r.work_max() == 8
        assert r.work_avg() == 4.0
    assert math.isclose(listed.work_stddev(), summed.work_stddev(), rel_tol=1e-12)
    assert math.isclose(listed.work_stddev(), float(np.std(work)), rel_tol=1e-12)


def test_verify_reports_first_mismatch():
    r = pkg.verify([0, 1, 2], [0, 1, 2])
    assert r.matched and r.mismatch_count == 0
    r = pkg.verify([0, 1, 2, 3], [0, 9, 2, 7])
    assert not r.matched and r.mismatch_count == 2 and r.first_mismatch == (1, 1, 9)


def test_run_strategy_validates_before_the_device():
    g = pkg.path_graph(4)
    with pytest.raises(ValueError):
        pkg.run_strategy("XX", g, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig())
    with pytest.raises(ValueError):
        pkg.run_strategy("bs", g, 4, pkg.RelaxOp("bfs"), pkg.KernelConfig())
    with pytest.raises(ValueError):
        pkg.run_ns(g, 0, pkg.RelaxOp("bfs"), pkg.KernelConfig(), mdt=0)
    assert pkg.STRATEGY_TAGS == ("BS", "EP", "WD", "NS", "HP")
    assert pkg.FALLBACK_TAG == "WD-fallback" and pkg.INFEASIBLE_MEMORY == "infeasible: memory"


def test_grid_generator_shape():
    g = pkg.grid_graph(5, seed=1)
    assert g.num_nodes == 25 and g.num_edges == 4 * 5 * 4  # 2k(k-1) undirected -> both ways
    deg = g.outdegrees().reshape(5, 5)
    assert deg[0, 0] == 2 and deg[0, 2] == 3 and deg[2, 2] == 4
    assert g.col_indices[g.row_offsets[12]:g.row_offsets[13]].tolist() == [7, 11, 13, 17]
    assert g.weights.min() >= 1 and g.weights.max() <= 255


def test_upload_narrowing_loops_match_numpy():
    """The AVX2 narrowing of the upload (glb_host_simd.cpp) against numpy,
    including unaligned tails and the range / byte checks."""
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    if not lib.glb_cpu_has_avx2():
        pytest.skip("host has no AVX2")
    f32 = lib.glb_narrow_u32_avx2
    f32.restype = ctypes.c_int
    f32.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_uint64]
    f8 = lib.glb_narrow_u8_avx2
    f8.restype = ctypes.c_uint64
    f8.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]
    rng = np.random.default_rng(5)
    for count in (0, 1, 7, 8, 9, 1000, 4099):
        src = rng.integers(0, 1000, size=count).astype(np.int64)
        dst = np.zeros(count + 64, dtype=np.uint32)
        d = dst[: count] if dst.ctypes.data % 32 == 0 else dst[8 - (dst.ctypes.data % 32) // 4:][:count]
        assert f32(src.ctypes.data, d.ctypes.data, count, 1000) == 0
        assert np.array_equal(d, src.astype(np.uint32))
        if count:
            bad = src.copy()
            bad[count // 2] = 1000
            assert f32(bad.ctypes.data, d.ctypes.data, count, 1000) != 0
            bad[count // 2] = -1
            assert f32(bad.ctypes.data, d.ctypes.data, count, 1000) != 0
        b = rng.integers(0, 256, size=count).astype(np.int64)
        d8 = np.zeros(count + 16, dtype=np.uint8)
        o = f8(b.ctypes.data, d8.ctypes.data, count)
        assert o == (int(np.bitwise_or.reduce(b)) if count else 0)
        assert np.array_equal(d8[:count], b.astype(np.uint8))
        if count:
            b[-1] = 300
            assert f8(b.ctypes.data, d8.ctypes.data, count) > 255
