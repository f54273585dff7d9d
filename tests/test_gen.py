"""Generator pins (SURVEY.md §8(c) 'Generator' row; App. A): closed-form n/nnz, Table 1
shape statistics (golden fixture), exact symmetry / Hermitian twist, stencil values, spectrum."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import gen
from tests import closed_form as cf

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_table1.json")


def to_scipy(m):
    n = len(m["row_ptr"]) - 1
    return sp.csr_matrix((m["values"], m["col_idx"], m["row_ptr"]), shape=(n, m["n"]))


@pytest.mark.parametrize("row", json.load(open(GOLD))["rows"], ids=lambda r: r["name"])
def test_table1_shapes(row):
    """n exact; nnz, mean and sd of row length within the App. A fit of PAPER.md T1."""
    spec = gen.CONFIGS[row["cfg"]]
    m = gen.make_matrix(spec)
    st = gen.row_stats(m["row_ptr"])
    assert st["n"] == row["n"]
    assert st["nnz"] == spec.nnz                              # closed form (App. A)
    assert abs(st["nnz"] - row["nnz"]) / row["nnz"] < 0.004    # App. A: ≤ 0.38 %
    assert abs(st["mean"] - row["mean"]) / row["mean"] < 0.004
    assert abs(st["sd"] - row["c9"]) / row["c9"] < 0.025       # c9 read as sd (L13), ≤ 2.1 %
    assert st["max"] == 27                                     # conforming hex: 27 (T1 Twingo 33/39 unreachable)
    # density column c5 = 100·nnz/n² (verified reading, L13)
    assert abs(100.0 * row["nnz"] / row["n"] ** 2 - row["density_pct"]) < 0.0015


def test_cube_closed_form():
    for N in (3, 7, 20):
        spec = gen.cube(N)
        m = gen.make_matrix(spec)
        assert m["n"] == N ** 3 and m["nnz"] == (3 * N - 2) ** 3
        lens = np.diff(m["row_ptr"])
        assert (lens == 27).sum() == (N - 2) ** 3


def test_stencil_entries():
    """Interior row values equal App. A's diagonal/face/edge/corner formulas."""
    spec = gen.BoxSpec(7, 6, 5, 0.1, 2.0, True, 0)
    eta = 0.05
    m = gen.make_matrix(spec, eta=eta)
    A = to_scipy(m)
    h, k2 = spec.h, spec.k ** 2
    z = 1 + 1j * eta
    want = {0: 8 * h / 3 - z * k2 * 8 * h ** 3 / 27, 1: -z * k2 * 2 * h ** 3 / 27,
            2: -h / 6 - z * k2 * h ** 3 / 54, 3: -h / 12 - z * k2 * h ** 3 / 216}
    i = 3 + 7 * (3 + 6 * 2)
    row = A.getrow(i)
    assert row.nnz == 27
    for c, v in zip(row.indices, row.data):
        dx, dy, dz = c % 7 - 3, (c // 7) % 6 - 3, c // 42 - 2
        nd = abs(dx) + abs(dy) + abs(dz)
        assert abs(v - want[nd]) <= 1e-15 * abs(want[0])
    # identity (shell) row
    assert A[0, 0] == pytest.approx(8 * h / 3, rel=0, abs=0) and A.getrow(0).nnz == 1


def test_symmetry_and_twist_hermitian():
    spec = gen.CONFIGS["C1"]
    A = to_scipy(gen.make_matrix(spec))
    assert abs(A - A.T).max() == 0.0                      # complex symmetric, exactly
    Ag = to_scipy(gen.make_matrix(spec, eta=0.0, twist_seed=gen.SEED_TWIST))
    assert abs(Ag - Ag.conj().T).max() == 0.0             # Hermitian, exactly (L9)
    off = (Ag - sp.diags(Ag.diagonal())).tocsr()
    off.eliminate_zeros()
    assert np.abs(off.data.imag).max() > 0.5 * np.abs(off.data).max()  # genuinely complex


def test_spectrum_dense():
    """Dense eigenvalues equal the closed form (App. A, 'checked 4.7e-15')."""
    spec = gen.BoxSpec(9, 7, 6, 0.2, 1.7, True, 3)
    eta = 0.05
    A = to_scipy(gen.make_matrix(spec, eta=eta)).toarray()
    ev = np.sort_complex(np.linalg.eigvals(A))
    lam = list(cf.box_eigs(spec, eta).ravel()) + [cf.ident_value(spec)] * (spec.n - np.prod(spec.free_dims))
    lam = np.sort_complex(np.array(lam))
    assert np.max(np.abs(ev - lam)) <= 1e-13 * np.max(np.abs(lam))


def test_row_range_slab_matches_full():
    spec = gen.BoxSpec(10, 9, 8, 0.1, 3.5, True, 5)
    full = gen.make_matrix(spec)
    r0, r1 = 137, 611
    part = gen.make_matrix(spec, row_range=(r0, r1))
    p0, p1 = full["row_ptr"][r0], full["row_ptr"][r1]
    assert np.array_equal(part["row_ptr"], full["row_ptr"][r0:r1 + 1] - p0)
    assert np.array_equal(part["col_idx"], full["col_idx"][p0:p1])
    assert np.array_equal(part["values"], full["values"][p0:p1])
    b = gen.make_rhs(full)
    bp = gen.make_rhs(part)
    assert np.array_equal(bp, b[r0:r1])


def test_random_csr_canonical():
    m = gen.random_csr(500, seed=3)
    rp, col = m["row_ptr"], m["col_idx"]
    lens = np.diff(rp)
    assert (lens == 0).any() and (lens == 1).any() and (lens > 32).any()
    for i in range(500):
        c = col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0)


def test_add_long_rows_stress_input():
    """NEXT-4 irregular-row stress input: Twingo's max row length 39 (PAPER.md T1), canonical
    CSR, every original entry kept, only the picked free rows grow."""
    m = gen.make_matrix("C2")
    s = gen.add_long_rows(m, frac=0.02, target_len=39)
    lens0, lens1 = np.diff(m["row_ptr"]), np.diff(s["row_ptr"])
    assert lens1.max() == 39 and np.all(lens1 >= lens0)
    grown = np.flatnonzero(lens1 > lens0)
    assert len(grown) == int(0.02 * m["free_mask"].sum()) and np.all(m["free_mask"][grown] == 1)
    for i in grown[:50]:
        c1 = s["col_idx"][s["row_ptr"][i]:s["row_ptr"][i + 1]]
        assert np.all(np.diff(c1) > 0)
        c0 = m["col_idx"][m["row_ptr"][i]:m["row_ptr"][i + 1]]
        v0 = m["values"][m["row_ptr"][i]:m["row_ptr"][i + 1]]
        v1 = s["values"][s["row_ptr"][i]:s["row_ptr"][i + 1]]
        assert np.array_equal(v1[np.searchsorted(c1, c0)], v0)
