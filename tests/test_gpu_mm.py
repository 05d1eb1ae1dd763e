"""§8f f1 on the GPU: load_matrix_market end to end (host parse, device
general fold + from_entries, device split) against the reference's golden
outcomes (tests/golden/mm.json, from oracle/_ref via make_golden.py mm) —
identical CSR or identical exception class and message."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "mm.json")))
CASES = {c["name"]: c for c in GOLD["cases"]}


def _write(tmp_path, name, body):
    p = tmp_path / f"{name}.mtx"
    with open(p, "w", newline="") as f:
        f.write(body)
    return str(p)


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_matrix_market_matches_reference(pb, tmp_path, name):
    g = CASES[name]
    p = _write(tmp_path, name, g["body"])
    if not g["ok"]:
        exc = ValueError if g["kind"] == 1 else pb.ExpmcError
        with pytest.raises(exc) as ei:
            pb.load_matrix_market(p)
        assert str(ei.value) == g["message"].replace("{path}", p)
        with pytest.raises(exc):
            pb.from_matrix_market(p)
        return
    c = pb.load_matrix_market(p)
    assert c.n == g["n"]
    assert c.row_ptr.tolist() == g["row_offset"]
    assert c.col.tolist() == g["neighbor"]
    assert [float(x).hex() for x in c.val] == g["weight"]
    assert [float(x).hex() for x in c.diag] == g["diag"]
    m = pb.from_matrix_market(p)
    s = m.export()
    np.testing.assert_array_equal(s["row_offset"], c.row_ptr)
    np.testing.assert_array_equal(s["weight"], c.val)


def _general_text(csr):
    out = ["%%MatrixMarket matrix coordinate real general", ""]
    cnt = 0
    for i in range(csr.n):
        if csr.diag[i] != 0.0:
            out.append(f"{i + 1} {i + 1} {float(csr.diag[i])!r}")
            cnt += 1
        for k in range(int(csr.row_ptr[i]), int(csr.row_ptr[i + 1])):
            out.append(f"{i + 1} {int(csr.col[k]) + 1} {float(csr.val[k])!r}")
            cnt += 1
    out[1] = f"{csr.n} {csr.n} {cnt}"
    return "\n".join(out) + "\n"


def test_matrix_market_roundtrip_split_is_bit_exact(pb, tmp_path):
    """write_matrix_market(BA graph with a diagonal) -> from_matrix_market:
    the device split equals split() of the original CSR bit for bit, for the
    symmetric file and for a general (both-triangle) file folded on the GPU."""
    csr = pb.gen_ba(20_000, 4, 1)
    rng = np.random.default_rng(3)
    csr.val[:] = 0.0
    # symmetric random weights: assign per undirected edge
    for i in range(csr.n):
        for k in range(int(csr.row_ptr[i]), int(csr.row_ptr[i + 1])):
            j = int(csr.col[k])
            if j > i:
                csr.val[k] = float(rng.integers(1, 1000)) / 7.0
    for i in range(csr.n):
        for k in range(int(csr.row_ptr[i]), int(csr.row_ptr[i + 1])):
            j = int(csr.col[k])
            if j < i:
                kk = int(csr.row_ptr[j]) + int(np.searchsorted(
                    csr.col[int(csr.row_ptr[j]):int(csr.row_ptr[j + 1])], i))
                csr.val[k] = csr.val[kk]
    csr.diag[::5] = -1.5
    want = pb.split(csr).export()
    sym = str(tmp_path / "ba.mtx")
    pb.write_matrix_market(csr, sym)
    gen = _write(tmp_path, "ba_general", _general_text(csr))
    for p in (sym, gen):
        got = pb.from_matrix_market(p).export()
        for k in ("row_offset", "neighbor", "weight", "cum", "rate", "d", "diag", "uniform_row"):
            np.testing.assert_array_equal(got[k], want[k], err_msg=f"{p}: {k}")


def test_general_fold_error_reports_first_sorted_pair(pb, tmp_path):
    csr = pb.gen_fd(2, 30, 1.0)
    text = _general_text(csr).splitlines()
    # break symmetry of two pairs; the reference reports the first in (row, col) order
    for k, ln in enumerate(text):
        if ln.startswith("500 501 "):
            text[k] = "500 501 2.0"
        if ln.startswith("12 13 "):
            text[k] = "12 13 3.0"
    p = _write(tmp_path, "broken", "\n".join(text) + "\n")
    with pytest.raises(pb.ExpmcError) as ei:
        pb.load_matrix_market(p)
    assert str(ei.value) == f"{p}:{len(text)}: general matrix is not symmetric at (12, 13)"
