"""Pins of the fp64 oracle (oracle/) against what the paper and mathematics fix (-m "not gpu").

Each test names the pin id of DESIGN.md §3.  None of these re-types the oracle's own loops:
the comparisons are against (a) values printed in the paper/SPEC (tests/golden), (b) the
paper's own described data flow written with numpy bmm/permute,
(c) closed forms and special cases that reduce to a textbook product, (d) brute force with
explicit 4-deep sums on tiny inputs, and (e) invariants (linearity, row independence).
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RTOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = np.linalg.norm(a - b)
    s = np.linalg.norm(b)
    return d / s if s > 0 else d


def rng_bf16ish(rng, *shape):
    """Random values exactly representable in bf16 (8-bit mantissa), like the real inputs."""
    x = rng.standard_normal(shape).astype(np.float32)
    u = x.view(np.uint32) & np.uint32(0xFFFF0000)
    return u.view(np.float32).astype(np.float64)


# ------------------------------------------------------------------------------ p1 -------------
def test_p1_blast_worked_example():
    g = json.load(open(os.path.join(GOLD, "blast_worked_example.json")))
    W = orc.blast_weight(g["V"], g["S"], g["U"])
    assert np.array_equal(W, np.array(g["W"]))
    # with X = I the forward product returns W itself
    Y = orc.blast_forward(np.eye(2), g["V"], g["S"], g["U"])
    assert np.array_equal(Y, np.array(g["W"]))


# ------------------------------------------------------------------------------ p2 -------------
@pytest.mark.parametrize("r", [1, 3, 8])
def test_p2_blast_b1_is_V_diag_s_U(r):
    """north_star: BLAST with b=1 equals U diag(s) V^T (paper orientation V diag(s) U)."""
    rng = np.random.default_rng(r)
    i, o, n = 7 * 8, 5 * 8, 9
    V, S, U, X = rng_bf16ish(rng, 1, i, r), rng_bf16ish(rng, 1, 1, r), rng_bf16ish(rng, 1, r, o), rng_bf16ish(rng, n, i)
    Wref = V[0] @ np.diag(S[0, 0]) @ U[0]
    assert rel(orc.blast_weight(V, S, U), Wref) < RTOL
    assert rel(orc.blast_forward(X, V, S, U), X @ Wref) < RTOL
    # s = 1 -> plain low rank
    ones = np.ones((1, 1, r))
    assert rel(orc.blast_forward(X, V, ones, U), orc.lowrank_forward(X, V[0], U[0])) < RTOL


# ------------------------------------------------------------------------------ p3 -------------
@pytest.mark.parametrize("b1,b2", [(2, 2), (3, 2), (2, 5), (4, 4)])
def test_p3_blast_S_ones_is_lowrank(b1, b2):
    """S == 1 for every block: W_{l,k} = V_l U_k is rank r overall."""
    rng = np.random.default_rng(b1 * 10 + b2)
    p, q, r, n = 8, 16, 8, 6
    V, U, X = rng_bf16ish(rng, b1, p, r), rng_bf16ish(rng, b2, r, q), rng_bf16ish(rng, n, b1 * p)
    S = np.ones((b1, b2, r))
    V_lr = V.reshape(b1 * p, r)                                 # [V_0; ...; V_{b1-1}]
    U_lr = np.concatenate([U[k] for k in range(b2)], axis=1)    # [U_0 ... U_{b2-1}]
    assert rel(orc.blast_forward(X, V, S, U), X @ V_lr @ U_lr) < RTOL


# ------------------------------------------------------------------------------ p4 -------------
@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
def test_p4_monarch_b1_is_lowrank(layout):
    rng = np.random.default_rng(4)
    i, o, rp, n = 24, 40, 8, 5
    V, U, X = rng_bf16ish(rng, 1, rp, i), rng_bf16ish(rng, 1, o, rp), rng_bf16ish(rng, n, i)
    ref = X @ V[0].T @ U[0].T
    assert rel(orc.monarch_forward(X, V, U, 1, 1, layout), ref) < RTOL
    assert rel(orc.monarch_weight(V, U, 1, 1, layout), V[0].T @ U[0].T) < RTOL


# ------------------------------------------------------------------------------ p5 -------------
@pytest.mark.parametrize("b1,b2,rp", [(2, 2, 3), (3, 2, 2), (2, 4, 1), (4, 3, 2)])
def test_p5_monarch_identity_blocks_is_permutation(b1, b2, rp):
    """Monarch with identity blocks is a pure permutation (north_star).  p = r' b2, q = b1 r',
    V[l] = I, U[k] = I -> Y[t, k q + l r' + rho] = X[t, l p + m(rho, k)] exactly."""
    p, q = rp * b2, b1 * rp
    V = np.stack([np.eye(rp * b2, p) for _ in range(b1)])
    U = np.stack([np.eye(q, b1 * rp) for _ in range(b2)])
    n = 3
    X = np.arange(n * b1 * p, dtype=np.float64).reshape(n, b1 * p) + 1.0
    for layout, m in ((orc.B2_FASTEST, lambda rho, k: rho * b2 + k),
                      (orc.RPRIME_FASTEST, lambda rho, k: k * rp + rho)):
        Y = orc.monarch_forward(X, V, U, b1, b2, layout)
        E = np.zeros_like(Y)
        for t, k, l, rho in itertools.product(range(n), range(b2), range(b1), range(rp)):
            E[t, k * q + l * rp + rho] = X[t, l * p + m(rho, k)]
        assert np.array_equal(Y, E), layout


def test_p5b_monarch_layout_golden():
    """The composite-index order of V's middle dim, SPEC.md L179 / PAPER.md L194-195."""
    g = json.load(open(os.path.join(GOLD, "monarch_layout_example.json")))
    b2, rp = g["b2"], g["r_blk"]
    # Identity-block Monarch with p = r' b2 exposes which (k, rho) each middle-dim row serves.
    for layout, key in ((orc.B2_FASTEST, "b2_fastest_order"), (orc.RPRIME_FASTEST, "rprime_fastest_order")):
        b1, p, q = 1, rp * b2, rp
        V = np.eye(rp * b2, p)[None]
        U = np.stack([np.eye(q, rp) for _ in range(b2)])
        X = np.eye(p)  # token t = one-hot on input feature t (= middle-dim row t)
        Y = orc.monarch_forward(X, V, U, b1, b2, layout)
        order = []
        for m in range(rp * b2):
            (col,) = np.nonzero(Y[m])[0]
            order.append([col // q, col % q])  # (k, rho)
        assert order == g[key]


# ------------------------------------------------------------------------------ p6 -------------
@pytest.mark.parametrize("b1,b2,rp", [(2, 2, 2), (3, 2, 1), (2, 3, 2)])
def test_p6_blast_reproduces_monarch(b1, b2, rp):
    """BLAST recovers Monarch by the choice of S: rank R = b1 b2 r' with
    S[l,k,(l',k',rho)] = delta_ll' delta_kk'."""
    rng = np.random.default_rng(b1 + 7 * b2 + 31 * rp)
    p, q, n = 8, 8, 4
    Vm, Um, X = rng_bf16ish(rng, b1, rp * b2, p), rng_bf16ish(rng, b2, q, b1 * rp), rng_bf16ish(rng, n, b1 * p)
    R = b1 * b2 * rp
    idx = lambda l, k, rho: (l * b2 + k) * rp + rho
    Vb = np.zeros((b1, p, R)); Sb = np.zeros((b1, b2, R)); Ub = np.zeros((b2, R, q))
    for l, k, rho in itertools.product(range(b1), range(b2), range(rp)):
        j = idx(l, k, rho)
        Vb[l, :, j] = Vm[l, rho * b2 + k, :]
        Sb[l, k, j] = 1.0
        Ub[k, j, :] = Um[k, :, l * rp + rho]
    assert rel(orc.blast_forward(X, Vb, Sb, Ub), orc.monarch_forward(X, Vm, Um, b1, b2)) < RTOL


# ------------------------------------------------------------------------------ p7 -------------
def _paper_monarch_flow(X, V, U, b1, b2, layout):
    """PAPER.md L194 data flow with numpy: bmm1 -> perm r'<->b2 -> perm b2<->b1 -> bmm2."""
    n = X.shape[0]
    R, p = V.shape[1], V.shape[2]
    rp = R // b2
    q = U.shape[1]
    Xb = X.reshape(n, b1, p).transpose(1, 0, 2)                  # (b1, n, p)
    Z = Xb @ V.transpose(0, 2, 1)                                # (b1, n, r' b2)
    if layout == orc.B2_FASTEST:
        Z = Z.reshape(b1, n, rp, b2).transpose(0, 1, 3, 2)       # r' <-> b2 -> (b1, n, b2, r')
    else:
        Z = Z.reshape(b1, n, b2, rp)                             # already r'-fastest (opt. 1)
    Z = Z.transpose(2, 1, 0, 3).reshape(b2, n, b1 * rp)          # b2 <-> b1 -> (b2, n, b1 r')
    Y = Z @ U.transpose(0, 2, 1)                                 # (b2, n, q)
    return Y.transpose(1, 0, 2).reshape(n, b2 * q)               # canonical k-major


def _paper_blast_flow(X, V, S, U):
    """PAPER.md L160 / Table 2 data flow: bmm1 -> S-weighted sum over l -> bmm2."""
    b1, p, r = V.shape
    b2, _, q = U.shape
    n = X.shape[0]
    Z = X.reshape(n, b1, p).transpose(1, 0, 2) @ V               # (b1, n, r)
    Zpp = np.einsum("lnr,lkr->knr", Z, S)                        # (b2, n, r)
    Y = Zpp @ U                                                  # (b2, n, q)
    return Y.transpose(1, 0, 2).reshape(n, b2 * q)


@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
@pytest.mark.parametrize("b1,b2,rp", [(2, 2, 2), (3, 4, 2), (4, 2, 3), (1, 3, 2)])
def test_p7_monarch_structured_eq_dense_eq_paper_flow(layout, b1, b2, rp):
    rng = np.random.default_rng(100 + b1 * 9 + b2 * 3 + rp + layout)
    p, q, n = 16, 8, 7
    V, U, X = rng_bf16ish(rng, b1, rp * b2, p), rng_bf16ish(rng, b2, q, b1 * rp), rng_bf16ish(rng, n, b1 * p)
    Ys = orc.monarch_forward(X, V, U, b1, b2, layout)
    Yd = orc.dense_forward(X, orc.monarch_weight(V, U, b1, b2, layout))
    Yp = _paper_monarch_flow(X, V, U, b1, b2, layout)
    assert rel(Ys, Yd) < RTOL and rel(Ys, Yp) < RTOL


@pytest.mark.parametrize("b1,b2,r", [(2, 2, 4), (3, 4, 8), (4, 2, 5), (1, 3, 2), (6, 6, 8)])
def test_p7_blast_structured_eq_dense_eq_paper_flow(b1, b2, r):
    rng = np.random.default_rng(200 + b1 * 9 + b2 * 3 + r)
    p, q, n = 8, 16, 5
    V, S, U = rng_bf16ish(rng, b1, p, r), rng_bf16ish(rng, b1, b2, r), rng_bf16ish(rng, b2, r, q)
    X = rng_bf16ish(rng, n, b1 * p)
    Ys = orc.blast_forward(X, V, S, U)
    Yd = orc.dense_forward(X, orc.blast_weight(V, S, U))
    Yp = _paper_blast_flow(X, V, S, U)
    assert rel(Ys, Yd) < RTOL and rel(Ys, Yp) < RTOL


def test_p7_lowrank_structured_eq_dense():
    rng = np.random.default_rng(7)
    V, U, X = rng_bf16ish(rng, 24, 8), rng_bf16ish(rng, 8, 40), rng_bf16ish(rng, 6, 24)
    assert rel(orc.lowrank_forward(X, V, U), orc.dense_forward(X, orc.lowrank_weight(V, U))) < RTOL
    assert rel(orc.lowrank_forward(X, V, U), X @ V @ U) < RTOL


# ------------------------------------------------------------------------------ p8 -------------
def _brute_blast(X, V, S, U):
    """Explicit 4-deep sum per output element from PAPER.md L64/L74:
    Y[t, k q + c] = sum_l sum_a X[t, l p + a] * sum_rho V_l[a,rho] S_{l,k}[rho] U_k[rho,c]."""
    b1, p, r = len(V), len(V[0]), len(V[0][0])
    b2, q = len(U), len(U[0][0])
    n = len(X)
    Y = [[0.0] * (b2 * q) for _ in range(n)]
    for t in range(n):
        for k in range(b2):
            for c in range(q):
                s = 0.0
                for l in range(b1):
                    for a in range(p):
                        for rho in range(r):
                            s += X[t][l * p + a] * V[l][a][rho] * S[l][k][rho] * U[k][rho][c]
                Y[t][k * q + c] = s
    return np.array(Y)


def _brute_monarch(X, V, U, b1, b2, layout):
    """Y[t, k q + c] = sum_l sum_a X[t, l p + a] sum_rho V_{l,k}[a,rho] U_{l,k}[rho,c]
     with V_{l,k}[a,rho] = V[l][m(rho,k)][a], U_{l,k}[rho,c] = U[k][c][l r'+rho]."""
    R, p = len(V[0]), len(V[0][0])
    rp = R // b2
    q = len(U[0])
    n = len(X)
    Y = [[0.0] * (b2 * q) for _ in range(n)]
    for t in range(n):
        for k in range(b2):
            for c in range(q):
                s = 0.0
                for l in range(b1):
                    for a in range(p):
                        for rho in range(rp):
                            m = rho * b2 + k if layout == orc.B2_FASTEST else k * rp + rho
                            s += X[t][l * p + a] * V[l][m][a] * U[k][c][l * rp + rho]
                Y[t][k * q + c] = s
    return np.array(Y)


@pytest.mark.parametrize("b1,b2", [(1, 1), (2, 3), (3, 2), (3, 3)])
def test_p8_brute_force_blast(b1, b2):
    rng = np.random.default_rng(300 + b1 * 5 + b2)
    p, q, r, n = 3, 2, 4, 3
    V, S, U = rng_bf16ish(rng, b1, p, r), rng_bf16ish(rng, b1, b2, r), rng_bf16ish(rng, b2, r, q)
    X = rng_bf16ish(rng, n, b1 * p)
    Yb = _brute_blast(X.tolist(), V.tolist(), S.tolist(), U.tolist())
    assert rel(orc.blast_forward(X, V, S, U), Yb) < 1e-13
    assert rel(orc.dense_forward(X, orc.blast_weight(V, S, U)), Yb) < 1e-13


@pytest.mark.parametrize("layout", [orc.B2_FASTEST, orc.RPRIME_FASTEST])
@pytest.mark.parametrize("b1,b2,rp", [(1, 1, 2), (2, 3, 1), (3, 2, 2)])
def test_p8_brute_force_monarch(layout, b1, b2, rp):
    rng = np.random.default_rng(400 + b1 * 5 + b2 + 17 * rp)
    p, q, n = 3, 2, 3
    V, U, X = rng_bf16ish(rng, b1, rp * b2, p), rng_bf16ish(rng, b2, q, b1 * rp), rng_bf16ish(rng, n, b1 * p)
    Yb = _brute_monarch(X.tolist(), V.tolist(), U.tolist(), b1, b2, layout)
    assert rel(orc.monarch_forward(X, V, U, b1, b2, layout), Yb) < 1e-13


# ------------------------------------------------------------------------------ p9 -------------
def test_p9_lowrank_identity_V_is_plain_gemm():
    rng = np.random.default_rng(9)
    i, o, n = 16, 24, 5
    X, U = rng_bf16ish(rng, n, i), rng_bf16ish(rng, i, o)
    assert rel(orc.lowrank_forward(X, np.eye(i), U), X @ U) < RTOL


# ------------------------------------------------------------------------------ p11 ------------
def test_p11_invariants_blast():
    rng = np.random.default_rng(11)
    b1, b2, p, q, r, n = 3, 2, 8, 8, 4, 6
    V, S, U = rng_bf16ish(rng, b1, p, r), rng_bf16ish(rng, b1, b2, r), rng_bf16ish(rng, b2, r, q)
    X1, X2 = rng_bf16ish(rng, n, b1 * p), rng_bf16ish(rng, n, b1 * p)
    f = lambda X: orc.blast_forward(X, V, S, U)
    # linearity in X
    assert rel(f(2.0 * X1 - 3.0 * X2), 2.0 * f(X1) - 3.0 * f(X2)) < 1e-12
    # row independence: permuting rows of X permutes rows of Y exactly
    perm = rng.permutation(n)
    assert np.array_equal(f(X1[perm]), f(X1)[perm])
    # zeroing S[l,k,:] zeroes block W_{l,k}
    S0 = S.copy(); S0[1, 0, :] = 0.0
    W = orc.blast_weight(V, S0, U)
    assert np.all(W[1 * p:2 * p, 0:q] == 0.0)
    assert np.any(W[0:p, 0:q] != 0.0)


def test_p11_monarch_relayout_invariance():
    """Re-layout (1) of V does not change the layer."""
    rng = np.random.default_rng(12)
    b1, b2, rp, p, q, n = 3, 4, 2, 8, 8, 5
    V, U, X = rng_bf16ish(rng, b1, rp * b2, p), rng_bf16ish(rng, b2, q, b1 * rp), rng_bf16ish(rng, n, b1 * p)
    # middle dim rho*b2 + k  ->  k*r' + rho
    Vr = V.reshape(b1, rp, b2, p).transpose(0, 2, 1, 3).reshape(b1, rp * b2, p)
    assert np.array_equal(orc.monarch_forward(X, V, U, b1, b2, orc.B2_FASTEST),
                          orc.monarch_forward(X, Vr, U, b1, b2, orc.RPRIME_FASTEST))


def test_oracle_empty_tokens():
    V, S, U = np.ones((2, 4, 2)), np.ones((2, 2, 2)), np.ones((2, 2, 4))
    Y = orc.blast_forward(np.zeros((0, 8)), V, S, U)
    assert Y.shape == (0, 8)


# ---------------------------------------------- transposed Monarch output order -----
def test_monarch_transposed_order_worked_example_and_identity_blocks():
    """Transposed order: b2 = 2 output blocks of q = 3 columns; canonical
    columns (k, c) = [00 01 02 10 11 12] appear as [00 10 01 11 02 12].  With identity blocks the
    whole layer is a closed-form integer permutation (pin p5 composed with the transposition)."""
    b1, b2, rp = 2, 2, 3
    p, q = rp * b2, b1 * rp
    V = np.stack([np.eye(rp * b2, p) for _ in range(b1)])
    U = np.stack([np.eye(q, b1 * rp) for _ in range(b2)])
    X = np.arange(2 * b1 * p, dtype=np.float64).reshape(2, b1 * p) + 1.0
    for layout in (orc.B2_FASTEST, orc.RPRIME_FASTEST):
        Yt = orc.monarch_forward_transposed(X, V, U, b1, b2, layout)
        for t in range(2):
            for k in range(b2):
                for l in range(b1):
                    for rho in range(rp):
                        a = rho * b2 + k if layout == orc.B2_FASTEST else k * rp + rho
                        c = l * rp + rho                     # canonical column inside block k
                        assert Yt[t, c * b2 + k] == X[t, l * p + a]
    # worked example, b1 = 1, b2 = 2, r' = q = 3, identity blocks, b2-fastest V rows (m = rho*b2 + k):
    # canonical Y[t, k*3 + c] = X[t, 2c + k] = X[:, [0, 2, 4, 1, 3, 5]], and the transposed order
    # Y[t, c*2 + k] = X[t, 2c + k] is X itself
    V1 = np.eye(6)[None]
    U1 = np.stack([np.eye(3), np.eye(3)])
    X1 = np.arange(12, dtype=np.float64).reshape(2, 6) + 1.0
    assert np.array_equal(orc.monarch_forward(X1, V1, U1, 1, 2), X1[:, [0, 2, 4, 1, 3, 5]])
    assert np.array_equal(orc.monarch_forward_transposed(X1, V1, U1, 1, 2), X1)


def test_transposed_output_chains_into_prepermuted_next_weight():
    """Optimization (3): Y_transposed @ W[perm] == Y_canonical @ W in fp64,
    with perm from the library's host helper (include/blr.h blr_transposed_row_perm)."""
    import paper_2512_20861_b200 as blr
    rng = np.random.default_rng(5)
    b1, b2, rp, p, q, n = 3, 4, 2, 5, 6, 7
    X = rng.standard_normal((n, b1 * p))
    V = rng.standard_normal((b1, rp * b2, p))
    U = rng.standard_normal((b2, q, b1 * rp))
    W2 = rng.standard_normal((b2 * q, 9))
    perm = blr.transposed_row_perm(b2, q).numpy()
    Yc = orc.monarch_forward(X, V, U, b1, b2)
    Yt = orc.monarch_forward_transposed(X, V, U, b1, b2)
    assert np.allclose(Yt @ W2[perm], Yc @ W2, rtol=1e-12, atol=1e-12)
    assert not np.allclose(Yt @ W2, Yc @ W2)
