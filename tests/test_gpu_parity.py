"""Device (C-ABI) vs CPU oracle parity on seeded inputs — the parity gate.

Bars: bit-exact for the integer index stream, gaussian_init and Jacobi (the
device Jacobi uses explicitly rounded intrinsics); floating point within the
tolerance written in each test (the device sums in a different order and with
FMA)."""
import numpy as np
import pytest

from oracle_lib import default_si_config
from problems import csc_to_dense, planted_dense, random_csc

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("seed,n,m", [(0, 5000, 5), (12345, 1, 7), (7, 2_000_000, 100_003), (2**63 + 5, 100_000, 1024),
                                      (99, 3, 513), (5, 1_000_000, 0)])
def test_index_stream_bit_exact(g, oracle, seed, n, m):
    dev = g.index_stream(seed, n, m)
    ref = oracle.uniform_index(seed, n, m).astype(np.int64)
    assert np.array_equal(dev.astype(np.int64), ref)


def test_index_stream_golden(g):
    # Rng(0).uniform_index(5000) x 5 = 1503 1255 4180 330 4874
    assert g.index_stream(0, 5000, 5).tolist() == [1503, 1255, 4180, 330, 4874]


def test_gaussian_init_bit_exact(g, oracle):
    for d, p, seed in [(4, 2, 0), (257, 7, 3), (1000, 10, 2**40)]:
        assert np.array_equal(g.gaussian_init(d, p, seed), oracle.gaussian_init(d, p, seed)[1])


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8, 10, 16, 20, 31, 32, 33, 64])
def test_gram_block_dense(g, oracle, p):
    rng = np.random.default_rng(p)
    d, n = 300, 1100
    X = rng.standard_normal((d, n))
    W = rng.standard_normal((d, p))
    x = g.DeviceMatrix.dense(X)
    z, y = g.gram_block(x, W, want_y=True)
    rc, zo, yo = oracle.gram_block(oracle.dense(X), W, want_y=True)
    assert rc == 0
    # |dZ| <= 1e-13 |X|^2 |W|
    scale = np.linalg.norm(X, 2) ** 2 * np.abs(W).max()
    assert np.abs(z - zo).max() <= 1e-13 * scale
    assert np.abs(y - yo).max() <= 1e-13 * np.linalg.norm(X, 2) * np.abs(W).max() * np.sqrt(d)


@pytest.mark.parametrize("d,n,p", [(4096, 3001, 20), (4096, 5, 1), (4096, 1000, 33), (2048, 4099, 32), (1000, 1601, 10),
                                   (1000, 777, 64), (300, 16, 2), (8192, 300, 3), (2050, 4099, 1), (1500, 1001, 1),
                                   (4096, 20001, 1), (1030, 3, 1), (8192, 301, 1), (6002, 999, 1)])
def test_gram_block_layouts(g, d, n, p):
    # every single-pass layout (16- / 8- / 4-CTA clusters, 256 / 128 rows per
    # CTA, ragged last tile, several clusters, 32-column chunks), the p = 1
    # single-pass kernels (1024 < d <= 8192: 2 / 4 / 8 rows per thread, w in
    # shared memory above 4096, odd n, fewer columns than CTAs) and the
    # two-pass fallback (d = 8192, p = 3) against a float64 numpy product
    rng = np.random.default_rng(d + n + p)
    X = rng.standard_normal((d, n))
    W = rng.standard_normal((d, p))
    z, y = g.gram_block(g.DeviceMatrix.dense(X), W, want_y=True)
    yr = X.T @ W
    zr = X @ yr
    scale = np.linalg.norm(X, 2) ** 2 * np.abs(W).max()
    assert np.abs(z - zr).max() <= 1e-13 * scale
    assert np.abs(y - yr).max() <= 1e-13 * np.linalg.norm(X, 2) * np.abs(W).max() * np.sqrt(d)


def test_gram_block_fused_forced_layouts(tmp_path):
    # the single-pass kernel is the default only for d <= 1024; force it
    # (GAPLRA_GRAM_FUSED=2, read once per process) for the 16- and 8-CTA
    # cluster layouts in a child process
    import os
    import subprocess
    import sys
    code = """
import sys, numpy as np
sys.path.insert(0, %r)
import paper_1607_02925_b200 as g
for d, n, p in [(4096, 3001, 20), (4096, 37, 1), (2048, 4099, 32), (4096, 999, 33)]:
    rng = np.random.default_rng(d + n + p)
    X = rng.standard_normal((d, n)); W = rng.standard_normal((d, p))
    z, y = g.gram_block(g.DeviceMatrix.dense(X), W, want_y=True)
    yr = X.T @ W; zr = X @ yr
    s = np.linalg.norm(X, 2)
    assert np.abs(z - zr).max() <= 1e-13 * s * s * np.abs(W).max(), (d, n, p)
    assert np.abs(y - yr).max() <= 1e-13 * s * np.abs(W).max() * np.sqrt(d), (d, n, p)
    assert np.array_equal(z, g.gram_block(g.DeviceMatrix.dense(X), W)), (d, n, p)
print("ok")
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GAPLRA_GRAM_FUSED="2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_gram_block_deterministic(g):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((512, 4096))
    W = rng.standard_normal((512, 20))
    x = g.DeviceMatrix.dense(X)
    a = g.gram_block(x, W)
    b = g.gram_block(x, W)
    assert np.array_equal(a, b)
    X = rng.standard_normal((2048, 5000))  # p = 1 single-pass kernel
    w = rng.standard_normal((2048, 1))
    x = g.DeviceMatrix.dense(X)
    assert np.array_equal(g.gram_block(x, w), g.gram_block(x, w))


def test_gram_apply_kats(g):
    # I3 (1,2,3) -> (1,2,3); diag(2,3) (1,1) -> (4,9)
    assert np.allclose(g.gram_apply(g.DeviceMatrix.dense(np.eye(3)), np.array([1.0, 2, 3])), [1, 2, 3], atol=0)
    assert np.allclose(g.gram_apply(g.DeviceMatrix.dense(np.diag([2.0, 3.0])), np.array([1.0, 1.0])), [4, 9], atol=0)


@pytest.mark.parametrize("p", [1, 4, 16])
def test_gram_block_sparse(g, oracle, p):
    d, n = 400, 3000
    cp, ri, v = random_csc(d, n, 20, seed=p)
    x = g.DeviceMatrix.csc(d, n, cp, ri, v)
    W = np.random.default_rng(0).standard_normal((d, p))
    z = g.gram_block(x, W)
    rc, zo, _ = oracle.gram_block(oracle.csc(d, n, cp, ri, v), W)
    assert rc == 0
    assert rel(z, zo) <= 1e-13


def test_qr_matches_oracle(g, oracle):
    rng = np.random.default_rng(3)
    for d, p in [(10, 4), (1000, 10), (4096, 20), (5000, 16), (9000, 12)]:
        y = rng.standard_normal((d, p))
        q = g.qr_orthonormalize(y)
        rc, qo, _ = oracle.qr(y)
        assert rc == 0
        assert rel(q, qo) <= 1e-12
        assert g.orthonormality_defect(q) <= 1e-12


def test_qr_rank_deficient(g):
    y = np.random.default_rng(0).standard_normal((50, 4))
    y[:, 2] = y[:, 0] + 2 * y[:, 1]
    with pytest.raises(g.RankDeficient) as e:
        g.qr_orthonormalize(y)
    assert e.value.column == 2
    with pytest.raises(g.RankDeficient) as e:
        g.qr_orthonormalize(np.zeros((5, 2)))
    assert e.value.column == 0


@pytest.mark.parametrize("n", [1, 2, 3, 10, 33, 64])
def test_jacobi_bit_exact(g, oracle, n):
    rng = np.random.default_rng(n)
    h = rng.standard_normal((n, n))
    h = h + h.T
    e = g.jacobi_eigh(h)
    rc, vals, vecs = oracle.jacobi(h)
    assert np.array_equal(e.values, vals)
    assert np.array_equal(e.vectors, vecs)


def test_jacobi_golden(g):
    e = g.jacobi_eigh(np.array([[4.0, 1, 0], [1, 3, 0], [0, 0, 1]]))
    assert e.values.tolist() == [4.6180339887498931, 2.3819660112501047, 1.0]


@pytest.mark.parametrize("p", [1, 3, 8, 20])
def test_svrg_epoch_lockstep(g, oracle, p):
    X, _, _ = planted_dense(64, 400, seed=p)
    rng = np.random.default_rng(p)
    lam = 1.05
    m = oracle.dense(X)
    w0 = rng.standard_normal((64, p))
    _, z, y = oracle.gram_block(m, w0, want_y=True)
    b = rng.standard_normal((64, p))
    eta = 1.0 / (4.0 * (lam + 400 * oracle.max_col_norm2(m)))
    cblk = eta * (z + b)
    rc, wo, idx = oracle.svrg_epoch(m, w0, y, cblk, eta, lam, 77, 800)
    wd = g.svrg_epoch(g.DeviceMatrix.dense(X), w0, y, cblk, eta, lam, 77, 800)
    assert rel(wd, wo) <= 1e-10


@pytest.mark.timeout(120)
@pytest.mark.parametrize("d,n,p,m", [
    (4096, 300, 1, 1000),   # 16-CTA clusters x 256 rows, warp-specialised chain, PC = 1
    (4096, 300, 3, 1000),   # PC = 3, one column group, two reducer warps
    (4096, 300, 20, 1000),  # C2 layout: tensor-core chain v4, 3 groups x PC 8 (last group 4 columns)
    (2048, 300, 32, 1000),  # C3 layout: v4 on 8-CTA clusters x 256 rows, 4 groups
    (4096, 300, 13, 1000),  # v4, ragged last group (5 columns)
    (1000, 300, 10, 1000),  # C1 layout (v3: d <= 1024)
    (8192, 200, 1, 500),    # C5 layout, p = 1: 512 rows per CTA (scalar chain)
    (8192, 200, 64, 500),   # C5 layout: PC 6, two waves of clusters (DMMA chain)
])
def test_svrg_epoch_lockstep_layouts(g, oracle, d, n, p, m):
    """One epoch at the production epoch layouts (m not a multiple of 16: a ragged last block)."""
    rng = np.random.default_rng(d + p)
    X = rng.standard_normal((d, n)) / np.sqrt(n)
    lam = 1.2 * np.linalg.norm(X, 2) ** 2
    mo = oracle.dense(X)
    w0 = rng.standard_normal((d, p))
    _, z, y = oracle.gram_block(mo, w0, want_y=True)
    eta = 1.0 / (4.0 * (lam + n * oracle.max_col_norm2(mo)))
    cblk = eta * (z + rng.standard_normal((d, p)))
    rc, wo, _ = oracle.svrg_epoch(mo, w0, y, cblk, eta, lam, 31, m)
    wd = g.svrg_epoch(g.DeviceMatrix.dense(X), w0, y, cblk, eta, lam, 31, m)
    assert rel(wd, wo) <= 1e-10


def test_svrg_epoch_sparse_lockstep(g, oracle):
    d, n, p = 120, 500, 4
    cp, ri, v = random_csc(d, n, 8, seed=2)
    m = oracle.csc(d, n, cp, ri, v)
    rng = np.random.default_rng(5)
    w0 = rng.standard_normal((d, p))
    _, z, y = oracle.gram_block(m, w0, want_y=True)
    lam = 2.0
    eta = 1.0 / (4.0 * (lam + n * oracle.max_col_norm2(m)))
    cblk = eta * (z + rng.standard_normal((d, p)))
    rc, wo, _ = oracle.svrg_epoch(m, w0, y, cblk, eta, lam, 9, 1000)
    wd = g.svrg_epoch(g.DeviceMatrix.csc(d, n, cp, ri, v), w0, y, cblk, eta, lam, 9, 1000)
    assert rel(wd, wo) <= 1e-10


@pytest.mark.timeout(120)
@pytest.mark.parametrize("d,n,z,p,m", [
    (5000, 20000, 20, 16, 40003),  # C4 density: 157 blocks of 256 steps, rare couplings
    (300, 2000, 12, 8, 6001),      # dense couplings: deep dependency levels within a block
    (40, 400, 20, 3, 997),         # row lists overflow: exact serial fallback per block
])
def test_svrg_epoch_sparse_blocked_lockstep(g, oracle, d, n, z, p, m):
    """Block-parallel sparse epoch (sparse_levels.cu) against the oracle's step-by-step epoch."""
    cp, ri, v = random_csc(d, n, z, seed=d + p)
    mo = oracle.csc(d, n, cp, ri, v)
    rng = np.random.default_rng(d)
    w0 = rng.standard_normal((d, p))
    _, zz, y = oracle.gram_block(mo, w0, want_y=True)
    lam = 1.5 * float(np.sum(v * v))  # ‖X‖_F² ≥ λ₁: a definite shift
    eta = 1.0 / (4.0 * (lam + n * oracle.max_col_norm2(mo)))
    cblk = eta * (zz + rng.standard_normal((d, p)))
    rc, wo, _ = oracle.svrg_epoch(mo, w0, y, cblk, eta, lam, 5, m)
    wd = g.svrg_epoch(g.DeviceMatrix.csc(d, n, cp, ri, v), w0, y, cblk, eta, lam, 5, m)
    assert rel(wd, wo) <= 1e-10


def test_svrg_epoch_sparse_dense_row_and_ragged(g, oracle):
    """Level-scheduled sparse epoch (sparse_levels.cu) on patterns outside its fast path: a row present in
    every column (its per-block list overflows: exact step-by-step fallback), and ragged columns incl. empty
    ones; p = 20 takes the warp-per-step variant."""
    rng = np.random.default_rng(17)
    d, n, m = 600, 1800, 2500
    cols = []
    for j in range(n):
        k = int(rng.integers(0, 9))  # 0..8 further rows: ragged, some columns hold only row 0
        rr = np.sort(rng.choice(np.arange(1, d), k, replace=False)) if k else np.zeros(0, np.int64)
        if j % 7 == 3:
            rows = rr  # a few columns without the dense row (possibly empty)
        else:
            rows = np.concatenate([[0], rr])
        cols.append(rows.astype(np.int32))
    cp = np.zeros(n + 1, np.int64)
    cp[1:] = np.cumsum([len(c) for c in cols])
    ri = np.concatenate(cols).astype(np.int32)
    v = rng.standard_normal(len(ri)) / np.sqrt(n)
    mo = oracle.csc(d, n, cp, ri, v)
    xs = g.DeviceMatrix.csc(d, n, cp, ri, v)
    lam = 1.5 * float(np.sum(v * v))
    eta = 1.0 / (4.0 * (lam + n * oracle.max_col_norm2(mo)))
    for p in (5, 20):
        w0 = rng.standard_normal((d, p))
        _, zz, y = oracle.gram_block(mo, w0, want_y=True)
        cblk = eta * (zz + rng.standard_normal((d, p)))
        _, wo, _ = oracle.svrg_epoch(mo, w0, y, cblk, eta, lam, 5, m)
        wd = g.svrg_epoch(xs, w0, y, cblk, eta, lam, 5, m)
        assert rel(wd, wo) <= 1e-10
        assert np.array_equal(wd, g.svrg_epoch(xs, w0, y, cblk, eta, lam, 5, m))


def test_svrg_epoch_sparse_many_rows(g, oracle):
    """d > 65536: the symbolic kernel keeps its row counters in global memory instead of shared memory."""
    d, n, z, p, m = 70000, 3000, 5, 3, 4001
    cp, ri, v = random_csc(d, n, z, seed=8)
    mo = oracle.csc(d, n, cp, ri, v)
    rng = np.random.default_rng(8)
    w0 = rng.standard_normal((d, p))
    _, zz, y = oracle.gram_block(mo, w0, want_y=True)
    lam = 1.5 * float(np.sum(v * v))
    eta = 1.0 / (4.0 * (lam + n * oracle.max_col_norm2(mo)))
    cblk = eta * (zz + rng.standard_normal((d, p)))
    _, wo, _ = oracle.svrg_epoch(mo, w0, y, cblk, eta, lam, 5, m)
    xs = g.DeviceMatrix.csc(d, n, cp, ri, v)
    wd = g.svrg_epoch(xs, w0, y, cblk, eta, lam, 5, m)
    assert rel(wd, wo) <= 1e-10
    # no steps: W = α Ŵ + β C with α = 1, β = 0
    assert np.array_equal(g.svrg_epoch(xs, w0, y, cblk, eta, lam, 5, 0), w0)


def test_svrg_epoch_sparse_older_kernels(tmp_path):
    """The fixed-point block kernel (GAPLRA_SPARSE_LEVELS=0) and the one-warp sequential kernel
    (GAPLRA_SPARSE_BLOCKED=0) stay selectable: same epoch against the oracle in child processes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = """
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1607_02925_b200 as g
from oracle_lib import Oracle
from problems import random_csc
o = Oracle()
d, n, z, p, m = 5000, 20000, 20, 16, 20011
cp, ri, v = random_csc(d, n, z, seed=3)
mo = o.csc(d, n, cp, ri, v)
rng = np.random.default_rng(1)
w0 = rng.standard_normal((d, p))
_, zz, y = o.gram_block(mo, w0, want_y=True)
lam = 1.5 * float(np.sum(v * v))
eta = 1.0 / (4.0 * (lam + n * o.max_col_norm2(mo)))
c = eta * (zz + rng.standard_normal((d, p)))
_, wo, _ = o.svrg_epoch(mo, w0, y, c, eta, lam, 5, m)
wd = g.svrg_epoch(g.DeviceMatrix.csc(d, n, cp, ri, v), w0, y, c, eta, lam, 5, m)
assert np.abs(wd - wo).max() <= 1e-10 * np.abs(wo).max()
print("ok")
""" % (root, os.path.join(root, "tests"))
    for extra in ({"GAPLRA_SPARSE_LEVELS": "0"}, {"GAPLRA_SPARSE_BLOCKED": "0"}):
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **extra), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, (extra, r.stdout + r.stderr)


def test_svrg_solve_matches_oracle_and_direct(g, oracle):
    X, _, sig = planted_dense(60, 300, seed=0)
    lam = 1.05
    b = np.random.default_rng(0).standard_normal((60, 3))
    r = g.solve_svrg(g.DeviceMatrix.dense(X), lam, b, 1e-10, seed=7)
    rc, wo, ep, hist = oracle.svrg_solve(oracle.dense(X), lam, b, 1e-10, seed=7)
    assert rc == 0
    assert abs(r.epochs - ep) <= 1
    assert rel(r.solution, wo) <= 1e-8
    wd = np.linalg.solve(lam * np.eye(60) - X @ X.T, b)
    assert rel(r.solution, wd) <= 1e-8


def test_svrg_solve_p1_single_pass_layout(g, oracle):
    # p = 1 at 1024 < d <= 4096: the anchor's gram pass and H = Xᵀ C take the
    # single-pass p = 1 kernel
    X, _, sig = planted_dense(1500, 2000, seed=3)
    lam = 1.05 * sig[0] ** 2
    b = np.random.default_rng(3).standard_normal((1500, 1))
    r = g.solve_svrg(g.DeviceMatrix.dense(X), lam, b, 1e-10, seed=5)
    rc, wo, ep, hist = oracle.svrg_solve(oracle.dense(X), lam, b, 1e-10, seed=5)
    assert rc == 0
    assert abs(r.epochs - ep) <= 1
    assert rel(r.solution, wo) <= 1e-8
    assert rel(r.solution, np.linalg.solve(lam * np.eye(1500) - X @ X.T, b)) <= 1e-8


def test_svrg_solve_zero_matrix(g):
    # X = 0, lambda = 1 -> x = b exactly after epoch 1
    b = np.arange(1.0, 9.0).reshape(8, 1)
    r = g.solve_svrg(g.DeviceMatrix.dense(np.zeros((8, 5))), 1.0, b, 1e-12)
    assert np.allclose(r.solution, b, rtol=1e-12)


def test_solver_stalls_on_indefinite_shift(g):
    X, _, _ = planted_dense(40, 200, seed=1)
    with pytest.raises(g.SolverStalled) as e:
        g.solve_svrg(g.DeviceMatrix.dense(X), 0.5, np.ones((40, 1)), 1e-10)
    assert len(e.value.residual_history) >= 1


def test_restricted_projection(g, oracle):
    X, U, sig = planted_dense(80, 200, seed=4)
    s = g.qr_orthonormalize(np.random.default_rng(1).standard_normal((80, 8)) + 3 * U[:, :8])
    w, ritz = g.restricted_projection(g.DeviceMatrix.dense(X), s, 4)
    rc, wo, ro = oracle.restricted_projection(oracle.dense(X), s, 4)
    assert rc == 0
    assert np.allclose(ritz, ro, rtol=1e-12)
    assert oracle.sin_theta(wo, w) <= 1e-10


def test_shift_invert_matches_oracle(g, oracle):
    from oracle_lib import default_si_config

    X, U, sig = planted_dense(60, 300, k=4, p=8, seed=0)
    lamv = sig ** 2
    delta = 2 / 3 * (lamv[3] - lamv[8])
    cfg = g.SIConfig(k=4, p=8, delta=delta, seed=5)
    res = g.shift_invert(g.DeviceMatrix.dense(X), cfg)
    rc, wo, ro, so, rep = oracle.shift_invert(oracle.dense(X), default_si_config(4, 8, delta=delta, seed=5))
    assert rc == 0
    assert res.lam == pytest.approx(rep.lambda_, rel=1e-10)
    assert res.tune_history and len(res.tune_history) == rep.tune_steps
    assert oracle.sin_theta(wo, res.W) <= 1e-8          # north star: sin theta <= 1e-8 (fp64)
    assert np.allclose(res.ritz, ro, rtol=1e-10)
    assert oracle.sin_theta(U[:, :4], res.W) <= 1e-8    # and against the planted truth
    assert abs(res.outer_iterations - rep.outer_iterations) <= 1


def test_shift_invert_sparse(g, oracle):
    from oracle_lib import default_si_config

    d, n = 100, 400
    cp, ri, v = random_csc(d, n, 8, seed=8, rank=3)
    Xd = csc_to_dense(d, n, cp, ri, v)
    ev = np.sort(np.linalg.eigvalsh(Xd @ Xd.T))[::-1]
    k, p = 2, 4
    lam = ev[0] + (ev[k - 1] - ev[p]) / 2
    cfg = g.SIConfig(k=k, p=p, lam=lam, seed=1, max_outer=40, conv_tol=1e-7)
    res = g.shift_invert(g.DeviceMatrix.csc(d, n, cp, ri, v), cfg)
    rc, wo, ro, so, rep = oracle.shift_invert(oracle.csc(d, n, cp, ri, v),
                                              default_si_config(k, p, lam=lam, seed=1, max_outer=40, conv_tol=1e-7))
    assert rc == 0
    assert oracle.sin_theta(wo, res.W) <= 1e-8
    assert np.allclose(res.ritz, ro, rtol=1e-10)
    assert np.allclose(res.ritz, ev[:k], rtol=1e-9)


# ---- solve_cg / error_report / principal_angles ----
@pytest.mark.parametrize("p", [1, 5, 20])
def test_cg_solve_matches_oracle_and_direct(g, oracle, p):
    X, _, sig = planted_dense(300, 900, seed=p)
    lam = sig[0] ** 2 * 1.02
    b = np.random.default_rng(p).standard_normal((300, p))
    r = g.solve_cg(g.DeviceMatrix.dense(X), lam, b, 1e-11)
    rc, wo, it, _ = oracle.cg_solve(oracle.dense(X), lam, b, 1e-11)
    assert rc == 0
    assert abs(r.epochs - it) <= 1
    assert rel(r.solution, wo) <= 1e-9
    assert rel(r.solution, np.linalg.solve(lam * np.eye(300) - X @ X.T, b)) <= 1e-9


def test_cg_solve_sparse_identity_and_indefinite(g):
    # D = I -> one iteration; lambda < lambda_1 -> IndefiniteShift
    b = np.random.default_rng(0).standard_normal((9, 2))
    r = g.solve_cg(g.DeviceMatrix.dense(np.zeros((9, 4))), 1.0, b, 1e-12)
    assert r.epochs == 1 and np.allclose(r.solution, b, atol=1e-15)
    X, U, sig = planted_dense(40, 80, seed=4)
    with pytest.raises(g.IndefiniteShift):
        g.solve_cg(g.DeviceMatrix.dense(X), 0.5 * sig[0] ** 2, U[:, :1] + 0.01, 1e-10)


def test_error_report_matches_oracle(g, oracle):
    X, U, sig = planted_dense(256, 700, seed=9, noise=1e-2)
    W, _ = np.linalg.qr(U[:, :4] + 1e-3 * np.random.default_rng(1).standard_normal((256, 4)))
    fd, sd = g.error_report(g.DeviceMatrix.dense(X), W, iters=30, seed=3)
    rc, fo, so = oracle.error_report(oracle.dense(X), W, iters=30, seed=3)
    assert rc == 0
    assert abs(fd - fo) <= 1e-12 * np.linalg.norm(X)
    assert abs(sd - so) <= 1e-10 * so
    assert abs(fd - np.linalg.norm(X - W @ (W.T @ X))) <= 1e-12 * np.linalg.norm(X)
    cp, ri, v = random_csc(200, 500, 7, seed=2)
    Xs = csc_to_dense(200, 500, cp, ri, v)
    Ws, _ = np.linalg.qr(np.random.default_rng(2).standard_normal((200, 3)))
    fd, sd = g.error_report(g.DeviceMatrix.csc(200, 500, cp, ri, v), Ws, iters=25, seed=5)
    rc, fo, so = oracle.error_report(oracle.csc(200, 500, cp, ri, v), Ws, iters=25, seed=5)
    assert abs(fd - fo) <= 1e-12 * np.linalg.norm(Xs) and abs(sd - so) <= 1e-10 * so


def test_principal_angles_matches_oracle(g, oracle):
    rng = np.random.default_rng(11)
    U, _ = np.linalg.qr(rng.standard_normal((500, 6)))
    S = U @ rng.standard_normal((6, 10)) + 1e-3 * rng.standard_normal((500, 10))
    cd = g.principal_angles(U, S)
    rc, co = oracle.principal_angles(U, S)
    assert rc == 0 and np.allclose(cd, co, atol=1e-13)
    Q, _ = np.linalg.qr(S)
    assert np.allclose(cd, np.linalg.svd(U.T @ Q, compute_uv=False), atol=1e-13)


def test_shift_invert_cg_backend(g, oracle):
    # inverse_operator(cg) in the pipeline: device vs oracle, and against the
    # svrg backend (Frobenius error within 1e-6 relative)
    X, U, sig = planted_dense(200, 1000, k=4, p=8, seed=12, noise=1e-3)
    lam = sig[0] ** 2 + 0.05
    x = g.DeviceMatrix.dense(X)
    kw = dict(k=4, p=8, lam=lam, seed=2, max_outer=80, lambda1_hint=sig[0] ** 2)
    rc_ = g.shift_invert(x, g.SIConfig(backend="cg", **kw))
    rs_ = g.shift_invert(x, g.SIConfig(**kw))
    rc, wo, ro, _, rep = oracle.shift_invert(
        oracle.dense(X), default_si_config(4, 8, lam=lam, seed=2, max_outer=80, hint=sig[0] ** 2, backend=1))
    assert rc == 0
    assert oracle.sin_theta(rc_.W, wo) <= 1e-8
    assert np.allclose(rc_.ritz, ro, rtol=1e-10)
    fc = g.error_report(x, rc_.W)[0]
    fs = g.error_report(x, rs_.W)[0]
    assert abs(fc - fs) <= 1e-6 * fs


# ---- Alg. 3 (k > 1), Alg. 4 / 5, Alg. 7 adaptive driver ----
def test_gap_detection_kats_device(g):
    assert g.detect_multiplicative_gap([4.0, 3.0, 2.99], 1, 2) == 1
    assert g.detect_multiplicative_gap([2.0, 2.0, 2.0], 1, 3) is None
    assert g.detect_multiplicative_gap([9.0, 8.9, 4.0], 4, 3) == 5
    assert g.detect_additive_gap([0.1, 0.2, 1.0], 2, 4, 1.0) == 3
    assert g.detect_additive_gap([0.1, 0.2, 0.3], 2, 4, 1.0) == 4
    with pytest.raises(g.ShiftOutOfRange):
        g.detect_additive_gap([0.5, 0.6], 1, 2, 1.0)


@pytest.mark.parametrize("k", [1, 3, 8])
def test_estimate_eigenvalues_matches_oracle(g, oracle, k):
    X, _, sig = planted_dense(200, 500, k=4, p=10, seed=20 + k, noise=1e-3)
    vd, itd = g.estimate_eigenvalues(g.DeviceMatrix.dense(X), k, 1 / 9, 7)
    rc, vo, ito = oracle.estimate_eigenvalues(oracle.dense(X), k, 1 / 9, 7)
    assert rc == 0 and abs(itd - ito) <= 1
    if itd == ito:
        assert np.allclose(vd, vo, rtol=1e-10)
    lam = np.linalg.eigvalsh(X @ X.T)[::-1][:k]
    assert np.all(vd >= (1 - 1 / 9) * lam - 1e-12) and np.all(vd <= lam / (1 - 1 / 9) + 1e-12)


def _check_approximate(g, oracle, X, cfg_kw, ocfg):
    x = g.DeviceMatrix.dense(X)
    res = g.approximate(x, g.SIConfig(**cfg_kw))
    rc, wo, ro, rep = oracle.approximate(oracle.dense(X), ocfg)
    assert rc == 0
    assert [(iv["s"], iv["q"], iv["strategy"], iv["width"]) for iv in res.plan] == \
        [(iv["s"], iv["q"], iv["strategy"], iv["width"]) for iv in rep.plan()]
    assert oracle.sin_theta(res.W, wo) <= 1e-7
    assert np.allclose(res.ritz, ro, rtol=1e-9)
    return res


def test_approximate_diag_device(g, oracle):
    X = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    res = _check_approximate(g, oracle, X, dict(k=2, p=4, eps=1e-3, delta=10.0, seed=1),
                             default_si_config(2, 4, eps=1e-3, delta=10.0, seed=1))
    assert res.frobenius_error <= (1 + 1e-3) * np.sqrt(14.0)


def test_approximate_shifted_inverse_device(g, oracle):
    sig = np.concatenate([[10.0, 9.99, 9.98, 5.0, 1.0], 0.5 / np.arange(1, 31)])
    X, U, _ = planted_dense(60, 80, sigma=sig, seed=11)
    gap = sig[2] ** 2 - sig[6] ** 2
    res = _check_approximate(g, oracle, X, dict(k=3, p=6, eps=1e-4, delta=gap / 1.5, seed=3, force=True,
                                                max_outer=400),
                             default_si_config(3, 6, eps=1e-4, delta=gap / 1.5, seed=3, force=1, max_outer=400))
    assert any(iv["strategy"] == "ShiftedInverse" and iv["s"] == 1 and iv["q"] >= 3 for iv in res.plan)
    assert res.frobenius_error <= (1 + 1e-4) * np.sqrt(np.sum(sig[3:] ** 2))


def test_approximate_deflated_intervals_device(g, oracle):
    # a multiplicative gap after index 1 and a small-gap tail: PlainPower {1}
    # then a deflated interval (CG on the deflated shifted system)
    sig = np.concatenate([[6.0, 3.0, 2.99, 2.98], 0.3 / np.arange(1, 41)])
    X, U, _ = planted_dense(80, 120, sigma=sig, seed=13)
    gap = sig[3] ** 2 - sig[6] ** 2
    res = _check_approximate(g, oracle, X, dict(k=4, p=7, eps=1e-4, delta=gap / 1.5, seed=4, force=True,
                                                max_outer=600),
                             default_si_config(4, 7, eps=1e-4, delta=gap / 1.5, seed=4, force=1, max_outer=600))
    assert len(res.plan) >= 2 and res.plan[0]["strategy"] == "PlainPower"
    assert res.frobenius_error <= (1 + 1e-4) * np.sqrt(np.sum(sig[4:] ** 2))


def test_find_gap_budget_device(g, oracle):
    X, U, sig = planted_dense(300, 800, k=5, p=10, seed=21, noise=1e-3)
    dd = g.find_gap_budget(g.DeviceMatrix.dense(X), 5, 10, seed=4)
    rc, do = oracle.find_gap_budget(oracle.dense(X), 5, 10, seed=4)
    assert rc == 0 and abs(dd - do) <= 1e-9 * do
    lam = sig ** 2
    assert dd <= lam[4] - lam[10] <= 2 * dd
    with pytest.raises(g.NoUsableGap):
        g.find_gap_budget(g.DeviceMatrix.dense(np.diag(np.sqrt([3.0, 2.0] + [1.0] * 8))), 3, 6, seed=1)


def test_approximate_auto_delta_device(g, oracle):
    X = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    res = _check_approximate(g, oracle, X, dict(k=2, p=3, eps=1e-3, delta=0.0, seed=1),
                             default_si_config(2, 3, eps=1e-3, delta=0.0, seed=1))
    assert 6.0 <= res.delta <= 12.0


def test_binary_x_to_device(g, tmp_path):
    # streamed binary X -> HBM (column chunks), same gram pass as the in-memory upload
    from paper_1607_02925_b200 import xio

    X, _, sig = planted_dense(301, 777, seed=5)
    xio.save_dense(tmp_path / "x.bin", X, sigma=sig.tolist())
    x, side = xio.load_dense_device(tmp_path / "x.bin")
    W = np.random.default_rng(0).standard_normal((301, 7))
    assert np.array_equal(g.gram_block(x, W), g.gram_block(g.DeviceMatrix.dense(X), W))
    assert side["sigma"] == sig.tolist()


def test_accelerated_svrg_device(g, oracle):
    X, U, sig = planted_dense(300, 900, seed=31)
    l1 = sig[0] ** 2
    lam = 1.02 * l1
    b = np.random.default_rng(3).standard_normal((300, 4))
    r = g.solve_accelerated_svrg(g.DeviceMatrix.dense(X), lam, b, 1e-10, lambda1_hint=l1, seed=2)
    rc, wo, ep, _ = oracle.accsvrg_solve(oracle.dense(X), lam, b, 1e-10, seed=2, hint=l1)
    assert rc == 0 and abs(r.epochs - ep) <= max(2, ep // 20)
    ref = np.linalg.solve(lam * np.eye(300) - X @ X.T, b)
    assert rel(r.solution, ref) <= 1e-8 and rel(r.solution, wo) <= 1e-8
    # inside the pipeline (backend accsvrg) the subspace matches the svrg backend's
    x = g.DeviceMatrix.dense(X)
    kw = dict(k=3, p=6, lam=l1 + 0.05, seed=2, max_outer=80, lambda1_hint=l1)
    ra = g.shift_invert(x, g.SIConfig(backend="accsvrg", **kw))
    rs_ = g.shift_invert(x, g.SIConfig(**kw))
    assert oracle.sin_theta(ra.W, rs_.W) <= 1e-7


def test_non_finite_inputs_rejected(g):
    """ContractViolation at the boundary, as the reference constructor / spmv
    do (sparse_matrix.cpp:29,70): non-finite X (checked on the device at
    creation), non-finite W / B, and a borrowed X with non-zero pad rows."""
    import torch

    X = np.random.default_rng(0).standard_normal((10, 7))
    X[3, 4] = np.nan
    with pytest.raises(g.ContractViolation):
        g.DeviceMatrix.dense(X)
    X[3, 4] = np.inf
    with pytest.raises(g.ContractViolation):
        g.DeviceMatrix.dense(X)
    X[3, 4] = 0.5
    x = g.DeviceMatrix.dense(X)
    w = np.ones((10, 2))
    w[1, 1] = np.nan
    with pytest.raises(g.ContractViolation):
        g.gram_block(x, w)
    with pytest.raises(g.ContractViolation):
        g.solve_svrg(x, 100.0, w, 1e-8)
    # borrowed device X: ld must be round_up(d, 4) and the pad rows zero
    xt = torch.zeros((7, 12), dtype=torch.float64, device="cuda")
    xt[:, :10] = torch.from_numpy(X.T.copy()).cuda()
    ok = g.DeviceMatrix.from_torch(xt, d=10)
    assert np.allclose(g.gram_block(ok, np.ones((10, 1))), X @ (X.T @ np.ones((10, 1))), rtol=1e-13)
    xt[2, 11] = 1.0
    with pytest.raises(g.ContractViolation):
        g.DeviceMatrix.from_torch(xt, d=10)
    xt2 = torch.zeros((7, 16), dtype=torch.float64, device="cuda")
    with pytest.raises(g.ContractViolation):
        g.DeviceMatrix.from_device(xt2.data_ptr(), 10, 7, 16, keep=xt2)


def test_approximate_exact_rank_k_device(g, oracle):
    """SPEC.md:541 exact-rank-k KAT on the device: the oversampled iterates are
    rank deficient and completed identically to the oracle."""
    from oracle_lib import default_si_config

    X, _, _ = planted_dense(40, 60, sigma=np.array([3.0, 2.0, 1.5]), seed=10)
    for delta in (1.5, 0.0):
        ap = g.approximate(g.DeviceMatrix.dense(X), g.SIConfig(k=3, p=6, eps=1e-6, delta=delta, seed=2))
        rc, wo, ro, rep = oracle.approximate(oracle.dense(X), default_si_config(3, 6, eps=1e-6, delta=delta, seed=2))
        assert rc == 0
        assert [(q["s"], q["q"], q["strategy"], q["width"]) for q in ap.plan] == \
               [(q["s"], q["q"], q["strategy"], q["width"]) for q in rep.plan()]
        assert np.linalg.norm(X - ap.W @ (ap.W.T @ X)) <= 1e-8 * np.linalg.norm(X)
        assert np.allclose(ap.ritz, ro, rtol=1e-10)
        assert oracle.sin_theta(wo, ap.W) <= 1e-8


def test_device_resident_epoch_loop(g, oracle):
    """North star item 5: a dense solve's epochs run on the device (CUDA-graph
    WHILE node, k_epoch_control): the host waits a fixed number of times per
    solve, not once per epoch, and the result, history and epoch count equal
    the oracle's host-driven loop."""
    X, _, sig = planted_dense(2048, 4000, seed=6)
    lam = 1.05 * sig[0] ** 2
    b = np.random.default_rng(6).standard_normal((2048, 4))
    x = g.DeviceMatrix.dense(X)
    ctx = x.ctx
    s0 = ctx.host_syncs()
    r = g.solve_svrg(x, lam, b, 1e-10, seed=3)
    syncs = ctx.host_syncs() - s0
    assert r.epochs >= 10
    assert syncs <= 6, (syncs, r.epochs)
    rc, wo, ep, hist = oracle.svrg_solve(oracle.dense(X), lam, b, 1e-10, seed=3)
    assert rc == 0 and abs(r.epochs - ep) <= 1
    assert rel(r.solution, wo) <= 1e-8
    n = min(len(hist), len(r.residual_history))
    assert np.allclose(r.residual_history[:n], hist[:n], rtol=1e-6)
