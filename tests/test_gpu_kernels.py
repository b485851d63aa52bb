"""Kernel-level parity on the B200: every fused kernel against the reference's
golden outputs (tests/golden, produced by the real pipekrylov) and against
the oracle at geometries the fixtures do not cover.  Bitwise."""

import numpy as np
import pytest

from oracle import pk_oracle as orc
from tests import golden_data as gd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1410_4054_b200 as pk

    return pk


@pytest.fixture(scope="module")
def fused(pk):
    from paper_1410_4054_b200 import fused

    return fused


def golden_setup(pk):
    f = gd.fused()
    a = pk.CsrMatrix(*gd.csr_arrays(f, "A"))
    v = {k.split("/")[1]: f[k] for k in f if k.startswith("vec/")}
    return f, a, v


@pytest.mark.parametrize("gi", range(6))
def test_fused_kernels_match_reference_golden(pk, fused, gi):
    f, a, v = golden_setup(pk)
    ng, gs = gd.manifest()["fused_geoms"][gi]
    ctx = pk.ExecutionContext(n_groups=ng, group_size=gs)
    key = f"g{gi}"
    q, part = fused.spmv_fused(a, dev(v["p"]), ("input", "result", dev(v["w"])), ctx)
    assert same(host(q), f[f"{key}/spmv/q"])
    assert same(host(part), f[f"{key}/spmv/part"])
    assert same(host(fused.spmv(a, dev(v["x"]), ctx)), f[f"{key}/spmv_plain"])

    x, r, p = dev(v["x"]), dev(v["r"]), dev(v["p"])
    part = fused.fused_cg_vector_update(x, r, p, dev(v["ap"]), 0.37, -0.8, ctx)
    for name, t in (("x", x), ("r", r), ("p", p), ("part", part)):
        assert same(host(t), f[f"{key}/cg/{name}"]), name

    rr0 = fused.reduce_stage1(dev(v["r"] * v["r0"]), ctx)
    assert same(host(rr0), f[f"{key}/bs/rr0"])
    s, spart, alpha = fused.fused_bicgstab_s_update(dev(v["r"]), dev(v["ap"]), dev(f[f"{key}/bs/rr0"]),
                                                    dev(f[f"{key}/bs/apr"]), ctx)
    assert same(host(s), f[f"{key}/bs/s"]) and same(host(spart), f[f"{key}/bs/part"])
    assert alpha == f[f"{key}/bs/alpha"][0]

    x, r, p = dev(v["x"]), dev(v["r"]), dev(v["p"])
    part = fused.fused_bicgstab_xrp_update(x, r, p, dev(v["s"]), dev(v["ap"]), dev(v["as"]), 0.3, 1.7, -0.4,
                                           dev(v["r0"]), ctx)
    for name, t in (("x", x), ("r", r), ("p", p), ("part", part)):
        assert same(host(t), f[f"{key}/xrp/{name}"]), name

    basis = [dev(v["b0"]), dev(v["b1"]), dev(v["b2"])]
    w = dev(v["v"])
    gpart = fused.fused_gs_stage1(basis, w, ctx)
    assert same(host(gpart), f[f"{key}/gs1/part"])
    coeffs, npart = fused.fused_gs_update(w, basis, gpart, ctx)
    assert same(host(coeffs), f[f"{key}/gsu/coeffs"]) and same(host(w), f[f"{key}/gsu/v"])
    assert same(host(npart), f[f"{key}/gsu/part"])
    nrm, xpart = fused.fused_gs_normalize(w, npart, dev(v["r"]), ctx)
    assert nrm == f[f"{key}/gsn/norm"][0]
    assert same(host(w), f[f"{key}/gsn/v"]) and same(host(xpart), f[f"{key}/gsn/part"])
    assert fused.dot(dev(v["x"]), dev(v["r"]), ctx) == f[f"{key}/dot"][0]


# geometries beyond the fixtures: k-chunk walks (G << n), wide groups with
# several leaves per thread (gs > 256), one element per lane, tails.
GEOMS = [(128, 256), (7, 64), (3, 2048), (64, 4096), (1, 1), (5, 8), (300, 1024), (2, 65536)]


@pytest.fixture(scope="module")
def big_system(pk):
    rng = np.random.default_rng(99)
    a, _ = pk.convdiff2d(301)  # n = 90601: tails everywhere
    n = a.n_rows
    vecs = {k: rng.standard_normal(n) for k in ("p", "w", "x", "r", "ap", "s", "as", "r0", "v", "b0", "b1", "b2", "b3", "b4")}
    return a, vecs


@pytest.mark.parametrize("geom", GEOMS)
def test_fused_kernels_match_oracle_at_many_geometries(pk, fused, big_system, geom):
    a, v = big_system
    if geom == (1, 1):
        pytest.skip("1x1 at n=90601 is covered by the golden tests at n=300")
    ctx = pk.ExecutionContext(n_groups=geom[0], group_size=geom[1])
    q, part = fused.spmv_fused(a, dev(v["p"]), ("input", "result", dev(v["w"]), "result"), ctx)
    oq, opart = orc.spmv_fused(a, v["p"], ("input", "result", v["w"], "result"), geom)
    assert same(host(q), oq) and same(host(part), opart)

    x, r, p = dev(v["x"]), dev(v["r"]), dev(v["p"])
    part = fused.fused_cg_vector_update(x, r, p, dev(v["ap"]), 0.37, -0.8, ctx)
    ox, orr, op = v["x"].copy(), v["r"].copy(), v["p"].copy()
    opart = orc.cg_update(ox, orr, op, v["ap"], 0.37, -0.8, geom)
    assert same(host(x), ox) and same(host(r), orr) and same(host(p), op) and same(host(part), opart)

    x, r, p = dev(v["x"]), dev(v["r"]), dev(v["p"])
    part = fused.fused_bicgstab_xrp_update(x, r, p, dev(v["s"]), dev(v["ap"]), dev(v["as"]), 0.3, 1.7, -0.4,
                                           dev(v["r0"]), ctx)
    ox, orr, op = v["x"].copy(), v["r"].copy(), v["p"].copy()
    opart = orc.bicg_xrp_update(ox, orr, op, v["s"], v["ap"], v["as"], 0.3, 1.7, -0.4, v["r0"], geom)
    assert same(host(x), ox) and same(host(r), orr) and same(host(p), op) and same(host(part), opart)

    names = ["b0", "b1", "b2", "b3", "b4"]
    basis = [dev(v[k]) for k in names]
    w = dev(v["v"])
    gpart = fused.fused_gs_stage1(basis, w, ctx)
    ogpart = orc.gs_stage1([v[k] for k in names], v["v"], geom)
    assert same(host(gpart), ogpart)
    coeffs, npart = fused.fused_gs_update(w, basis, gpart, ctx)
    ow = v["v"].copy()
    oc, onpart = orc.gs_update(ow, [v[k] for k in names], ogpart, geom)
    assert same(host(coeffs), oc) and same(host(w), ow) and same(host(npart), onpart)
    nrm, xpart = fused.fused_gs_normalize(w, npart, dev(v["r"]), ctx)
    onrm, oxpart = orc.gs_normalize(ow, onpart, v["r"], geom, 1e-30)
    assert nrm == onrm and same(host(w), ow) and same(host(xpart), oxpart)


def test_spmv_fused_known_answer(pk, fused):
    # test_fused.py:59-67: [[4,1],[1,3]] @ [1,2] = [6,7]; <q,p> = 20, <q,q> = 85
    a = pk.CsrMatrix.from_dense([[4.0, 1.0], [1.0, 3.0]])
    q, part = fused.spmv_fused(a, dev([1.0, 2.0]), ("input", "result"), pk.ExecutionContext(2, 4))
    assert host(q).tolist() == [6.0, 7.0]
    tot = host(fused.reduce_stage2(part, pk.ExecutionContext(2, 4)))
    assert tot.tolist() == [20.0, 85.0]


def test_breakdown_flags(pk, fused):
    ctx = pk.ExecutionContext(1, 1)
    with pytest.raises(fused.BreakdownError):
        fused.fused_bicgstab_s_update(dev([1.0]), dev([1.0]), dev([[1.0]]), dev([[0.0]]), ctx)
    with pytest.raises(fused.LuckyBreakdown):
        z = dev([0.0, 0.0])
        fused.fused_gs_normalize(z, dev([[0.0]]), dev([1.0, 0.0]), ctx)


def test_stage1_known_answer(pk, fused):
    part = fused.reduce_stage1(dev(np.ones(1024)), pk.ExecutionContext(4, 256))
    assert host(part)[:, 0].tolist() == [256.0] * 4


def test_long_rows_take_the_remainder_path(pk, fused):
    # rows longer than the register window (8) and empty rows
    rng = np.random.default_rng(4)
    dense = rng.standard_normal((400, 400))
    dense[rng.random((400, 400)) > 0.08] = 0.0
    dense[17] = 0.0
    a = pk.CsrMatrix.from_dense(dense)
    assert a.row_nnz().max() > 8
    p = rng.standard_normal(400)
    for geom in [(128, 256), (3, 16)]:
        q, part = fused.spmv_fused(a, dev(p), ("input", "result"), pk.ExecutionContext(*geom))
        oq, opart = orc.spmv_fused(a, p, ("input", "result"), geom)
        assert same(host(q), oq) and same(host(part), opart)


@pytest.mark.gpu
def test_vec_update_kinds_bitwise():
    """pk_vec_update: every kind equals the reference's NumPy expression
    (linalg.py:403-457, solvers.py:277-280, 477-482) bit for bit, including
    signed zeros, subnormals and non-finite inputs."""
    import ctypes as C

    import torch

    import paper_1410_4054_b200 as pk
    from paper_1410_4054_b200 import _native as N
    from paper_1410_4054_b200.device import context_for

    rng = np.random.default_rng(12)
    n = 100_003
    y0, x, z = (rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n) for _ in range(3))
    for v in (y0, x, z):
        v[:8] = [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1.0]
    a, bta = -0.3712, 1.9e3
    want = {
        N.VEC_AXPY: y0 + a * x,
        N.VEC_AXPY2: y0 + (a * x + bta * z),
        N.VEC_XPAY: y0 * bta + x,
        N.VEC_SCALE: y0 * a,
        N.VEC_ADD_SCALED: x + a * z,
        N.VEC_BICG_P: (y0 - bta * z) * a + x,
        N.VEC_COPY: x.copy(),
    }
    ctx = pk.ExecutionContext()
    dc = context_for(ctx)
    dc.set_stream(torch.cuda.current_stream())
    xd, zd = torch.from_numpy(x).cuda(), torch.from_numpy(z).cuda()
    with np.errstate(all="ignore"):
        for kind, ref in want.items():
            yd = torch.from_numpy(y0.copy()).cuda()
            N.check(N.lib().pk_vec_update(dc.handle, kind, n, C.c_void_p(yd.data_ptr()), C.c_void_p(xd.data_ptr()),
                                          C.c_void_p(zd.data_ptr()), a, bta), "vec")
            got = yd.cpu().numpy()
            assert np.array_equal(got.view(np.int64)[~np.isnan(ref)], ref.view(np.int64)[~np.isnan(ref)]), kind
            assert np.array_equal(np.isnan(got), np.isnan(ref)), kind


@pytest.mark.parametrize("geom", [(16, 64), (4, 256), (1, 1024), (8, 32), (2, 4096)])
def test_spmv_fused_empty_and_long_rows(pk, fused, geom):
    """Rows with no entries and rows longer than the kernels' slot count (the
    remainder path), on short lane chains (2 <= K <= 8: the pipelined lane
    engine) and others; CSR and SELL-32 walks vs the oracle, bitwise."""
    rng = np.random.default_rng(3)
    n = 5000
    lens = rng.integers(0, 12, n)
    lens[rng.random(n) < 0.1] = 0
    lens[::97] = 40
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens])
    vals = rng.standard_normal(rows.size)
    a = pk.CsrMatrix.from_coo(n, n, rows, cols, vals)
    p, w = rng.standard_normal(n), rng.standard_normal(n)
    ctx = pk.ExecutionContext(*geom)
    oq, opart = orc.spmv_fused(a, p, ("input", "result", w), geom)
    for fmt in ("csr", "sell32"):
        dm = pk.DeviceMatrix.upload(pk.context_for(ctx), a).set_format(fmt, ctx)
        q, part = fused.spmv_fused(dm, dev(p), ("input", "result", dev(w)), ctx)
        assert same(host(q), oq) and same(host(part), opart), fmt


@pytest.mark.parametrize("geom", [(16, 64), (4, 256), (128, 256), (2, 4096)])
def test_spmv_fused_vec_rows(pk, fused, geom):
    """Long-row matrix (avg >= 24 entries per row): the SpMV row sums come
    from the warp-cooperative VEC pre-pass (k_rowsum_warp) and the fused
    operator runs as an elementwise reduction over them -- bitwise vs the
    oracle, with empty rows, a 700-entry row and rows longer than 32."""
    rng = np.random.default_rng(11)
    n = 3000
    lens = rng.integers(10, 50, n)
    lens[rng.random(n) < 0.05] = 0
    lens[7] = 700
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens])
    vals = rng.standard_normal(rows.size)
    a = pk.CsrMatrix.from_coo(n, n, rows, cols, vals)
    assert a.nnz >= 24 * n
    p, w = rng.standard_normal(n), rng.standard_normal(n)
    ctx = pk.ExecutionContext(*geom)
    oq, opart = orc.spmv_fused(a, p, ("input", "result", w), geom)
    dm = pk.DeviceMatrix.upload(pk.context_for(ctx), a)
    q, part = fused.spmv_fused(dm, dev(p), ("input", "result", dev(w)), ctx)
    assert same(host(q), oq) and same(host(part), opart)
    assert same(host(fused.spmv_csr(dm, dev(p), ctx)), oq)  # plain SpMV: VEC pre-pass + elementwise sweep
