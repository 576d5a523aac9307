"""Equilibration + static pivoting and Matrix Market ingestion (SURVEY §8f
row 3): bit-exact with the reference (oracle/_ref) and the reference's own
known-answer cases (test_sparse_core.cpp:181-232, 293-377) restated."""
import os

import numpy as np
import pytest

import paper_1502_07405_b200 as P


def csr(n, trip):
    """SparseMatrix::from_triplets semantics through a Matrix Market file is
    exercised below; here: duplicates summed, rows sorted (small KATs)"""
    d = {}
    for i, j, v in trip:
        d[(i, j)] = d.get((i, j), 0.0) + v
    ptr, ind, val = [0], [], []
    for i in range(n):
        row = sorted((j, v) for (r, j), v in d.items() if r == i)
        ind += [j for j, _ in row]
        val += [v for _, v in row]
        ptr.append(len(ind))
    return P.SparseMatrix.from_csr(n, np.array(ptr, np.int32), np.array(ind, np.int32),
                                   np.array(val, np.float64))


def badly_scaled(n, seed):
    rng = np.random.default_rng(seed)
    trip = []
    for i in range(n):
        rs = 10.0 ** ((i % 7) - 3)
        off = 0.0
        for d in (-5, -1, 2, 9):
            j = i + d
            if 0 <= j < n:
                v = rng.uniform(-1, 1)
                off += abs(v)
                trip.append((i, j, rs * v))
        trip.append((i, i, rs * (off + 1.0)))
    return csr(n, trip)


def permuted_unsym(n, seed):
    # a random column permutation of a diagonally dominant matrix: the
    # matching has to find the permutation back
    rng = np.random.default_rng(seed)
    q = rng.permutation(n)
    trip = []
    for i in range(n):
        trip.append((i, int(q[i]), 10.0 ** rng.uniform(-4, 4)))
        for j in rng.integers(0, n, 3):
            trip.append((i, int(j), rng.uniform(-1e-3, 1e-3)))
    return csr(n, trip)


def dense(a):
    ptr, ind, val = a.arrays()
    n = a.size()
    out = np.zeros((n, n))
    for i in range(n):
        out[i, ind[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
    return out


def test_hollow_2x2_goes_onto_a_unit_diagonal():
    # test_sparse_core.cpp:293-309
    a = csr(2, [(0, 1, 2.0), (1, 0, 3.0)])
    s, st = P.equilibrate_and_permute(a)
    assert list(st.qc) == [1, 0] and st.sweeps >= 1
    ds, da = dense(s), dense(a)
    assert ds[0, 0] == pytest.approx(1.0) and ds[1, 1] == pytest.approx(1.0)
    for i in range(2):
        for j in range(2):
            assert ds[i, j] == pytest.approx(st.dr[i] * da[i, st.qc[j]] * st.dc[st.qc[j]])


def test_badly_scaled_maxima_land_in_range_and_solve_roundtrips():
    # test_sparse_core.cpp:311-361
    n = 24
    a = badly_scaled(n, 99)
    s, st = P.equilibrate_and_permute(a)
    ds = dense(s)
    assert np.all((np.abs(ds).max(1) >= 0.5) & (np.abs(ds).max(1) <= 2.0))
    assert np.all((np.abs(ds).max(0) >= 0.5) & (np.abs(ds).max(0) <= 2.0))
    assert np.all(np.diag(ds) != 0.0)
    xt = np.random.default_rng(3).uniform(-1, 1, n)
    b = dense(a) @ xt
    xs = np.linalg.solve(ds, st.apply_scaling(b))
    assert np.allclose(st.undo_scaling(xs), xt, rtol=1e-9, atol=1e-12)


def test_structural_singularity_is_detected(oracle):
    # test_sparse_core.cpp:363-377
    for n, trip in [(2, [(0, 0, 1.0), (0, 1, 1.0)]),
                    (3, [(0, 2, 1.0), (1, 2, 1.0), (2, 0, 1.0), (2, 1, 1.0), (2, 2, 1.0)])]:
        a = csr(n, trip)
        with pytest.raises(P.StructuralSingularError):
            P.equilibrate_and_permute(a)
        with pytest.raises(oracle.RefError):
            oracle.equilibrate(*a.arrays())


def test_equilibration_bit_exact(oracle):
    mats = [badly_scaled(24, 99), badly_scaled(500, 4), permuted_unsym(300, 5),
            permuted_unsym(2000, 6), P.generate_convdiff3d(8, 0.1).A,
            P.generate_grid_problem("c2d", 20, 1e-3).A, P.generate_grid_problem("p3d", 6).A]
    for a in mats:
        s, st = P.equilibrate_and_permute(a)
        oi, ov, dr, dc, qc, sw = oracle.equilibrate(*a.arrays())
        ptr, ind, val = s.arrays()
        assert np.array_equal(ptr, a.arrays()[0])
        assert np.array_equal(ind, oi) and val.tobytes() == ov.tobytes()
        assert st.dr.tobytes() == dr.tobytes() and st.dc.tobytes() == dc.tobytes()
        assert np.array_equal(st.qc, qc) and st.sweeps == sw


def test_matrix_market_roundtrip_preserves_every_bit(tmp_path):
    # test_sparse_core.cpp:181-193
    a = csr(4, [(0, 0, 2.0), (0, 2, -1.0), (1, 1, 3.0), (1, 0, 0.5), (2, 2, 4.0), (2, 3, 1.5),
                (3, 3, 5.0), (0, 2, -0.5)])
    p = str(tmp_path / "rt.mtx")
    P.write_matrix_market(a, p)
    b = P.read_matrix_market(p)
    for x, y in zip(a.arrays(), b.arrays()):
        assert x.tobytes() == y.tobytes()
    a2 = badly_scaled(200, 8)
    P.write_matrix_market(a2, p)
    for x, y in zip(a2.arrays(), P.read_matrix_market(p).arrays()):
        assert x.tobytes() == y.tobytes()


def test_matrix_market_symmetric_and_duplicates_bit_exact(oracle, tmp_path):
    # test_sparse_core.cpp:195-213, plus duplicates summed in sorted order and
    # integer fields, against the reference reader
    p = str(tmp_path / "sym.mtx")
    with open(p, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n% comment line\n3 3 4\n"
                "1 1 2\n2 1 -1\n3 2 -1\n3 3 2\n")
    a = P.read_matrix_market(p)
    d = dense(a)
    assert a.nnz() == 6 and d[0, 1] == -1 and d[1, 0] == -1 and d[1, 2] == -1 and d[1, 1] == 0
    rng = np.random.default_rng(2)
    lines = [f"{rng.integers(1, 41)} {rng.integers(1, 41)} {rng.uniform(-1, 1)!r}"
             for _ in range(400)]
    for sym, field in [("general", "real"), ("symmetric", "real"), ("general", "integer")]:
        body = lines if field == "real" else [" ".join(x.split()[:2]) + f" {k % 7 - 3}"
                                              for k, x in enumerate(lines)]
        with open(p, "w") as f:
            f.write(f"%%MatrixMarket matrix coordinate {field} {sym}\n40 40 {len(body)}\n")
            f.write("\n".join(body) + "\n")
        mine = P.read_matrix_market(p).arrays()
        ref = oracle.read_mm(p)
        for x, y in zip(mine, ref):
            assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("text", [
    "%%NotMatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\nx y z\n",
])
def test_matrix_market_reader_rejects_malformed_files(tmp_path, text):
    # test_sparse_core.cpp:215-232
    p = str(tmp_path / "bad.mtx")
    with open(p, "w") as f:
        f.write(text)
    with pytest.raises(P.IoError):
        P.read_matrix_market(p)


def test_missing_file_is_an_io_error(tmp_path):
    with pytest.raises(P.IoError):
        P.read_matrix_market(os.path.join(str(tmp_path), "no_such_file.mtx"))
