"""GPU parity of the gradient oracle (kr_engine C ABI) against the CPU oracle.

The engine accumulates every output row in the reference's storage order
(engine.hpp:67-70, 82-88, 104-108, 118-129) with contraction disabled, so the
bar here is BITWISE equality with the oracle's matvec/matvecTranspose — the
north star's 1e-12 relative tolerance is asserted too, as the weaker
statement.  Factors come from the product's host builder (libkrhost), the
oracle's own factors are used to cross-check that path."""
import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal
from paper_2112_03804_b200 import ContractError, CudaEngine, InvalidInputError
from paper_2112_03804_b200 import host as H

pytestmark = pytest.mark.gpu

TOL = 1e-12  # north star: matvec outputs within 1e-12 relative (normwise, solver.hpp:87-88)


def normwise(got, exp):
    return np.abs(got - exp).max() / (1 + np.abs(exp).max())


def corpus():
    out = [(n, {}) for n in ("golden", "twenty_card", "bluffing", "all_tie")]
    out += [("random_small", dict(seed=s)) for s in range(8)]
    out += [("bench", dict(seed=2, hands=100))]
    return out


def check_engine(eng, sp, rows, cols, rng, trials=3):
    for _ in range(trials):
        x, y = rng.standard_normal(cols), rng.standard_normal(rows)
        ax, ex = eng.Ax(x), sp.matvec(x)
        aty, ey = eng.ATx(y), sp.matvec_t(y)
        assert normwise(ax, ex) <= TOL and normwise(aty, ey) <= TOL
        assert bits_equal(ax, ex) and bits_equal(aty, ey)


@pytest.mark.parametrize("name,kw", corpus())
@pytest.mark.parametrize("tech", ["a", "b"])
@pytest.mark.parametrize("post", [False, True])
def test_products_bitwise(name, kw, tech, post):
    p = H.builtin(name, **kw)
    o = po.Instance.builtin(name, **kw)
    eng = CudaEngine(p.sparsify(tech, post))
    check_engine(eng, o.sparsify(tech, post), p.rows, p.cols, np.random.default_rng(17))


@pytest.mark.parametrize("comp", [False, True], ids=["sell", "sell_c"])
@pytest.mark.parametrize("board,v", [("Ks7d4c2h9s", 3390846), ("AhKhQh7c7d", 2049828)], ids=["dry", "wet"])
def test_config2_products_bitwise(board, v, comp, monkeypatch):
    """Config 2 on the dry board and the wet one SURVEY.md §8(d) also names,
    with plain and compressed (KR_SELL_COMP) slots."""
    if comp:
        monkeypatch.setenv("KR_SELL_COMP", "1")
    p = H.builtin("river_full", seed=1, board=board, tree=3)
    o = po.Instance.builtin("river_full", seed=1, board=board, tree=3)
    eng = CudaEngine(p.sparsify("b", True))
    assert eng.nnz == {"ahat": 2754388, "u": 61617, "m": 62697, "v": v}
    check_engine(eng, o.sparsify("b", True), p.rows, p.cols, np.random.default_rng(3), trials=2)


def test_config2_technique_a_bitwise():
    """Config 2 through Technique A (the peel hits its rank cap of 1000, so
    U and V carry the low-rank term at full size)."""
    p = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    o = po.Instance.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    eng = CudaEngine(p.sparsify("a", True))
    assert eng.nnz == {"ahat": 9666364, "u": 795578, "m": 29028, "v": 795578}
    check_engine(eng, o.sparsify("a", True), p.rows, p.cols, np.random.default_rng(9), trials=1)


def test_config4_technique_a_bitwise():
    p = H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
    o = po.Instance.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
    eng = CudaEngine(p.sparsify("a", True))
    assert eng.m_identity
    check_engine(eng, o.sparsify("a", True), p.rows, p.cols, np.random.default_rng(4), trials=2)


def test_matches_dense_and_block_formula():
    """test_engine.cpp:38-64 on the GPU: vs the dense A and referenceMatvec(T)."""
    o = po.Instance.builtin("random_small", seed=9)
    A = o.dense()
    scale = 1 + np.abs(A).max()
    for tech in ("a", "b"):
        eng = CudaEngine(H.builtin("random_small", seed=9).sparsify(tech, True))
        x = np.random.default_rng(0).uniform(-1, 1, o.cols)
        y = np.random.default_rng(1).uniform(-1, 1, o.rows)
        assert np.abs(eng.Ax(x) - A @ x).max() < 1e-9 * scale
        assert np.abs(eng.ATx(y) - A.T @ y).max() < 1e-9 * scale
        assert np.abs(eng.Ax(x) - o.reference_matvec(x)).max() < 1e-9 * scale
        assert np.abs(eng.ATx(y) - o.reference_matvec_t(y)).max() < 1e-9 * scale


def test_deterministic_repeats_and_flops():
    """test_engine.cpp:66-77 (bitwise repeats) and 133-157 (flop counter)."""
    f = H.builtin("twenty_card").sparsify("b", True)
    eng = CudaEngine(f)
    x = np.random.default_rng(5).standard_normal(f.cols)
    first = eng.Ax(x)
    for _ in range(3):
        assert bits_equal(eng.Ax(x), first)
    per = f.nnz["v"] + f.nnz["u"] + f.nnz["ahat"] + f.nnz["m"] - f.k
    assert eng.last_flops() == per == 54925
    assert eng.flops() == 4 * per
    eng.ATx(np.ones(f.rows))
    assert eng.flops() == 5 * per
    a = CudaEngine(H.builtin("twenty_card").sparsify("a", False))
    a.Ax(np.ones(a.cols))
    assert a.last_flops() == a.nnz["v"] + a.nnz["u"] + a.nnz["ahat"]


def test_errors_mirror_the_reference():
    """test_engine.cpp:105-131: wrong sizes -> INVALID_INPUT; bad M -> CONTRACT."""
    f = H.builtin("golden").sparsify("b", False)
    eng = CudaEngine(f)
    with pytest.raises(InvalidInputError):
        eng.Ax(np.zeros(3))
    with pytest.raises(InvalidInputError):
        eng.ATx(np.zeros(3))
    arr = f.factors()
    k = f.k
    scaled = (np.arange(k + 1, dtype=np.int64), np.arange(k, dtype=np.int32), np.full(k, 2.0))
    bad = CudaEngine(dict(arr, rows=f.rows, cols=f.cols, k=k, m=scaled))
    with pytest.raises(ContractError):
        bad.Ax(np.ones(f.cols))
    # an entry above the diagonal: column 5 starts with row 0
    outer = np.concatenate([np.arange(6), np.arange(7, k + 2)]).astype(np.int64)
    inner = np.concatenate([np.arange(5), [0, 5], np.arange(6, k)]).astype(np.int32)
    above = (outer, inner, np.concatenate([np.ones(5), [0.25, 1.0], np.ones(k - 6)]))
    with pytest.raises(ContractError):
        CudaEngine(dict(arr, rows=f.rows, cols=f.cols, k=k, m=above)).ATx(np.ones(f.rows))


def test_general_unit_lower_m_level_schedule():
    """A random unit-lower M (test_engine.cpp:79-103 style) takes the level-
    scheduled solve path; results stay bitwise equal to the oracle."""
    rng = np.random.default_rng(17)
    f = H.builtin("random_small", seed=2).sparsify("b", False)
    arr = f.factors()
    k = f.k
    cols = []
    for j in range(k):
        rows = [j] + sorted(i for i in range(j + 1, k) if rng.uniform() < 0.05)
        cols.append((rows, [1.0] + list(rng.uniform(-1, 1, len(rows) - 1))))
    outer = np.cumsum([0] + [len(r) for r, _ in cols]).astype(np.int64)
    inner = np.concatenate([r for r, _ in cols]).astype(np.int32)
    val = np.concatenate([v for _, v in cols])
    arr["m"] = (outer, inner, val)
    eng = CudaEngine(dict(arr, rows=f.rows, cols=f.cols, k=k))
    osp = po.Sparsification.from_arrays(f.rows, f.cols, k, arr)
    check_engine(eng, osp, f.rows, f.cols, rng)


def test_multiboard_engine_matches_per_board():
    boards = H.turn_instances(nboards=4)
    eng = CudaEngine([f for _, f in boards])
    rng = np.random.default_rng(8)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ax, aty = eng.Ax(x), eng.ATx(y)
    r0 = c0 = 0
    for inst, f in boards:
        single = CudaEngine(f)
        assert bits_equal(ax[r0:r0 + inst.rows], single.Ax(x[c0:c0 + inst.cols]))
        assert bits_equal(aty[c0:c0 + inst.cols], single.ATx(y[r0:r0 + inst.rows]))
        r0 += inst.rows
        c0 += inst.cols


def test_device_pointer_entry_points():
    import torch
    f = H.builtin("twenty_card").sparsify("b", True)
    eng = CudaEngine(f)
    x = torch.randn(f.cols, dtype=torch.float64, device="cuda")
    y = torch.empty(f.rows, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    eng.ax_device(x.data_ptr(), y.data_ptr())
    torch.cuda.ExternalStream(eng.stream).synchronize()
    assert bits_equal(y.cpu().numpy(), eng.Ax(x.cpu().numpy()))


@pytest.mark.parametrize("groups,knob", [("1", None), ("2", None), ("3", None), ("4", None), ("4", ("KR_LPT", "0")),
                                         ("3", ("KR_LPT_ALL", "1")), ("2", ("KR_PF", "2")),
                                         ("3", ("KR_SELL_COMP", "1")), ("4", ("KR_ORDER", "sm")),
                                         ("4", ("KR_XSEQ", "1")), ("4", ("KR_PIPE_STREAMS", "2")),
                                         ("4", ("KR_GROUP_SIZES", "1,2,1"))])
def test_host_pipeline_groups_bitwise(groups, knob, monkeypatch):
    """kr_engine_ax / kr_engine_atx pipelined over board groups (each group's
    whole product on two streams, widest slices first) give the bits of the
    oracle, under every dispatch-order and prefetch variant."""
    monkeypatch.setenv("KR_GROUPS", groups)
    if knob:
        monkeypatch.setenv(*knob)
    ps = [H.builtin("river_full", seed=10 + k, board=b, deck=26, tree=3)
          for k, b in enumerate(["Kc9d7c4d2c", "Ac8d6c3d2d", "QcJd9c5d3c", "Tc7d5c4d2c"])]
    os_ = [po.Instance.builtin("river_full", seed=10 + k, board=b, deck=26, tree=3)
           for k, b in enumerate(["Kc9d7c4d2c", "Ac8d6c3d2d", "QcJd9c5d3c", "Tc7d5c4d2c"])]
    eng = CudaEngine([p.sparsify("b", True) for p in ps])
    sps = [o.sparsify("b", True) for o in os_]
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ax, aty = eng.Ax(x), eng.ATx(y)
    cx = np.cumsum([0] + [p.cols for p in ps])
    cy = np.cumsum([0] + [p.rows for p in ps])
    ex = np.concatenate([sp.matvec(x[cx[b]:cx[b + 1]]) for b, sp in enumerate(sps)])
    ey = np.concatenate([sp.matvec_t(y[cy[b]:cy[b + 1]]) for b, sp in enumerate(sps)])
    assert bits_equal(ax, ex) and bits_equal(aty, ey)


@pytest.mark.parametrize("serial_gb", [None, "0"], ids=["concurrent", "serial"])
@pytest.mark.parametrize("kind", ["factored", "implicit", "device_built"])
def test_pair_device_is_bitwise_ax_then_atx(kind, serial_gb, monkeypatch):
    """kr_engine_pair_device (A^T y forked onto a side stream, own scratch)
    gives the bits of kr_engine_ax_device then kr_engine_atx_device, also
    when repeated back to back on the same buffers."""
    import torch
    boards = H.turn_instances(nboards=3, factors=kind == "factored")
    if kind == "factored":
        eng = CudaEngine([f for _, f in boards])
    elif kind == "implicit":
        eng = CudaEngine.kron([i for i, _ in boards])
    else:
        eng = CudaEngine.device_built([i for i, _ in boards])
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax, atx = torch.empty(eng.rows, dtype=torch.float64, device="cuda"), torch.empty(eng.cols, dtype=torch.float64,
                                                                                     device="cuda")
    ax2, atx2 = torch.empty_like(ax), torch.empty_like(atx)
    torch.cuda.synchronize()
    eng.ax_device(x.data_ptr(), ax.data_ptr())
    eng.atx_device(y.data_ptr(), atx.data_ptr())
    for _ in range(3):
        eng.pair_device(x.data_ptr(), ax2.data_ptr(), y.data_ptr(), atx2.data_ptr())
    torch.cuda.ExternalStream(eng.stream).synchronize()
    assert torch.equal(ax, ax2) and torch.equal(atx, atx2)


@pytest.mark.parametrize("no_graph", [False, True], ids=["graph", "enqueued"])
@pytest.mark.parametrize("kind", ["factored", "implicit"])
def test_pinned_host_calls_replay_a_graph_bitwise(kind, no_graph, monkeypatch):
    """kr_engine_ax / kr_engine_atx on pinned host buffers: the first call
    enqueues the pipeline, the second captures it into a CUDA graph, later
    calls replay it; every call returns the bits of the device-pointer path,
    also after the input buffer's contents change (the graph reads the
    buffer, not a snapshot) and with a second pair of buffers."""
    import ctypes

    import torch
    from paper_2112_03804_b200 import _native as N
    if no_graph:
        monkeypatch.setenv("KR_NO_PIPE_GRAPH", "1")
    boards = H.turn_instances(nboards=3, factors=kind == "factored")
    eng = CudaEngine([f for _, f in boards]) if kind == "factored" else CudaEngine.kron([i for i, _ in boards])
    L = N.cuda()
    nx, ny = eng.cols, eng.rows
    arr = lambda p, n: np.ctypeslib.as_array((ctypes.c_double * n).from_address(p))  # noqa: E731
    bufs = [(L.kr_host_alloc(8 * nx), L.kr_host_alloc(8 * ny)) for _ in range(2)]
    try:
        rng = np.random.default_rng(21)
        for call in range(5):
            px, py = bufs[call % 2 if call >= 3 else 0]
            x = rng.standard_normal(nx)
            arr(px, nx)[:] = x
            N.check(L.kr_engine_ax(eng.handle, px, nx, py, ny))
            dx = torch.from_numpy(x).cuda()
            dy = torch.empty(ny, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            eng.ax_device(dx.data_ptr(), dy.data_ptr())
            torch.cuda.ExternalStream(eng.stream).synchronize()
            assert bits_equal(arr(py, ny).copy(), dy.cpu().numpy()), call
    finally:
        for px, py in bufs:
            L.kr_host_free(px)
            L.kr_host_free(py)


def test_host_call_after_async_device_call_is_ordered():
    """A host-buffer call issued while a device-pointer product is still in
    flight on the engine stream forks its pipeline streams from that stream
    (evStart), so neither call sees the other's scratch (d_tz / d_tz2)."""
    import torch
    boards = H.turn_instances(nboards=4)
    eng = CudaEngine([f for _, f in boards])
    rng = np.random.default_rng(31)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ref_ax, ref_atx = eng.Ax(x), eng.ATx(y)
    dx = torch.from_numpy(rng.standard_normal(eng.cols)).cuda()
    dy = torch.from_numpy(rng.standard_normal(eng.rows)).cuda()
    oax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    oatx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(3):
        eng.ax_device(dx.data_ptr(), oax.data_ptr())      # queued, not waited for
        eng.atx_device(dy.data_ptr(), oatx.data_ptr())
        got_ax, got_atx = eng.Ax(x), eng.ATx(y)           # host calls right behind
        assert bits_equal(got_ax, ref_ax) and bits_equal(got_atx, ref_atx)
    torch.cuda.ExternalStream(eng.stream).synchronize()
    assert bits_equal(oax.cpu().numpy(), eng.Ax(dx.cpu().numpy()))
    assert bits_equal(oatx.cpu().numpy(), eng.ATx(dy.cpu().numpy()))


@pytest.mark.parametrize("kind,nb", [("factored", 1), ("factored", 4), ("implicit", 4), ("kfactored", 4),
                                     ("kfactored", 1)])
def test_host_pair_call_bitwise(kind, nb):
    """kr_engine_pair (both directions' copies and kernels in flight together)
    gives the bits of kr_engine_ax then kr_engine_atx, on pageable buffers and
    on pinned ones (enqueued, captured, then replayed as a graph), also after
    the inputs change."""
    import ctypes

    from paper_2112_03804_b200 import _native as N
    boards = H.turn_instances(nboards=nb, factors=kind == "factored")
    insts = [i for i, _ in boards]
    eng = (CudaEngine([f for _, f in boards]) if kind == "factored" else
           CudaEngine.kron(insts) if kind == "implicit" else CudaEngine.kfactored(insts))
    rng = np.random.default_rng(41)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ax, atx = eng.pair(x, y)
    assert bits_equal(ax, eng.Ax(x)) and bits_equal(atx, eng.ATx(y))
    L = N.cuda()
    arr = lambda p, n: np.ctypeslib.as_array((ctypes.c_double * n).from_address(p))  # noqa: E731
    ptrs = [L.kr_host_alloc(8 * n) for n in (eng.cols, eng.rows, eng.rows, eng.cols)]
    try:
        px, py, pax, patx = (arr(p, n) for p, n in zip(ptrs, (eng.cols, eng.rows, eng.rows, eng.cols)))
        for call in range(4):
            px[:], py[:] = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
            N.check(L.kr_engine_pair(eng.handle, ptrs[0], eng.cols, ptrs[2], eng.rows, ptrs[1], eng.rows, ptrs[3],
                                     eng.cols))
            assert bits_equal(pax.copy(), eng.Ax(px.copy())), call
            assert bits_equal(patx.copy(), eng.ATx(py.copy())), call
    finally:
        for p in ptrs:
            L.kr_host_free(p)
    with pytest.raises(InvalidInputError):
        eng.pair(x[:-1], y)


@pytest.mark.parametrize("kind,nb", [("factored", 1), ("factored", 4), ("implicit", 4), ("kfactored", 4)])
def test_pair_queue_bitwise(kind, nb):
    """kr_engine_pair_queue: every queued pair's results are the bits of
    kr_engine_pair on it — on pageable and pinned buffers, with a buffer
    shared by several queue entries, for queues of 1, 2 and 5 pairs (slot
    reuse from the third pair on)."""
    import ctypes

    from paper_2112_03804_b200 import _native as N
    boards = H.turn_instances(nboards=nb, factors=kind == "factored")
    insts = [i for i, _ in boards]
    eng = (CudaEngine([f for _, f in boards]) if kind == "factored" else
           CudaEngine.kron(insts) if kind == "implicit" else CudaEngine.kfactored(insts))
    rng = np.random.default_rng(43)
    for q in (1, 2, 5):
        xs = [rng.standard_normal(eng.cols) for _ in range(q)]
        ys = [rng.standard_normal(eng.rows) for _ in range(q)]
        axs, atxs = eng.pair_queue(xs, ys)
        for i in range(q):
            ax, atx = eng.pair(xs[i], ys[i])
            assert bits_equal(axs[i], ax) and bits_equal(atxs[i], atx), (q, i)
    L = N.cuda()
    arr = lambda p, n: np.ctypeslib.as_array((ctypes.c_double * n).from_address(p))  # noqa: E731
    sizes = (eng.cols, eng.rows, eng.rows, eng.cols)
    bufs = [[L.kr_host_alloc(8 * n) for n in sizes] for _ in range(3)]
    try:
        for b in bufs:
            arr(b[0], eng.cols)[:] = rng.standard_normal(eng.cols)
            arr(b[1], eng.rows)[:] = rng.standard_normal(eng.rows)
        order = [0, 1, 2, 0, 1, 2, 2]   # entries share buffers; the last writer of an output is its last entry
        P = ctypes.c_void_p * len(order)
        col = lambda j: P(*[bufs[o][j] for o in order])  # noqa: E731
        N.check(L.kr_engine_pair_queue(eng.handle, len(order), col(0), eng.cols, col(2), eng.rows, col(1), eng.rows,
                                       col(3), eng.cols))
        for b in bufs:
            ax, atx = eng.pair(arr(b[0], eng.cols).copy(), arr(b[1], eng.rows).copy())
            assert bits_equal(arr(b[2], eng.rows).copy(), ax) and bits_equal(arr(b[3], eng.cols).copy(), atx)
    finally:
        for b in bufs:
            for p in b:
                L.kr_host_free(p)
    with pytest.raises(InvalidInputError):
        eng.pair_queue([rng.standard_normal(eng.cols + 1)], [rng.standard_normal(eng.rows)])
    assert eng.pair_queue([], []) == ([], [])


@pytest.mark.parametrize("name,kw", [("twenty_card", {}), ("bench", dict(seed=2, hands=100)),
                                     ("river_full", dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3))])
@pytest.mark.parametrize("tech", ["a", "b"])
def test_deep_batches_bitwise(name, kw, tech, monkeypatch):
    """Small grids run the SELL kernels with 16 entries per lane per batch
    (kr_engine.cu deep_batches): the same storage-order sums as the 8-entry
    kernels (KR_DEEP_KU=0), bit for bit, on both directions."""
    p = H.builtin(name, **kw)
    sp = p.sparsify(tech, True)
    rng = np.random.default_rng(23)
    x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
    monkeypatch.setenv("KR_TINY", "0")
    deep = CudaEngine(sp)
    a1, b1 = deep.Ax(x), deep.ATx(y)
    monkeypatch.setenv("KR_DEEP_KU", "0")
    plain = CudaEngine(sp)
    a0, b0 = plain.Ax(x), plain.ATx(y)
    assert bits_equal(a1, a0) and bits_equal(b1, b0)
