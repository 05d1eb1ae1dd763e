"""§8f rows f1 (Matrix Market I/O) and f3 (binary CSR cache), host side.

Parity with load_matrix_market / write_matrix_market
(proj/src/matrix_market.cpp:51-207) is pinned two ways:
  * tests/golden/mm.json — outcomes of the compiled reference on every case
    of tests/mm_cases.py (messages with the path as ``{path}``) and the
    reference writer's text for small matrices (make_golden.py mm);
  * the live reference (oracle/_ref) on larger generated files, when built.
The parse runs on the host (all cores); the general fold + from_entries run
on the GPU and are covered in tests/test_gpu_parity.py.  Here the fold is
restated in numpy (test-side) to check the parsed entries end to end.
"""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "mm.json")))
CASES = {c["name"]: c for c in GOLD["cases"]}


def _write(tmp_path, name, body):
    p = tmp_path / f"{name}.mtx"
    with open(p, "w", newline="") as f:
        f.write(body)
    return str(p)


def _fold_and_check(pb, e, path):
    """Test-side restatement of the rest of load_matrix_market after the
    parse: general fold (matrix_market.cpp:136-164) then from_entries'
    checks (sparse_matrix.cpp:20-51).  Returns ("ok", canonical entries) or
    (kind, message)."""
    r, c, w = e.rows.astype(np.int64), e.cols.astype(np.int64), e.weights
    if e.general:
        lo, hi = np.minimum(r, c), np.maximum(r, c)
        order = np.lexsort((hi, lo))
        lo, hi, ws = lo[order], hi[order], w[order]
        keep_r, keep_c, keep_w = [], [], []
        k = 0
        while k < len(lo):
            run = 1
            while k + run < len(lo) and lo[k + run] == lo[k] and hi[k + run] == hi[k]:
                run += 1
            if lo[k] == hi[k]:
                if run != 1:
                    return 2, f"{path}:{e.last_line}: duplicate diagonal entry ({lo[k] + 1}, {hi[k] + 1})"
            elif run != 2 or ws[k] != ws[k + 1]:
                return 2, f"{path}:{e.last_line}: general matrix is not symmetric at ({lo[k] + 1}, {hi[k] + 1})"
            keep_r.append(lo[k]); keep_c.append(hi[k]); keep_w.append(ws[k])
            k += run
        r, c, w = np.array(keep_r, np.int64), np.array(keep_c, np.int64), np.array(keep_w)
    for k in range(len(w)):
        at = f"({r[k]}, {c[k]})"
        if not np.isfinite(w[k]):
            return 1, f"non-finite weight at {at}"
        if w[k] == 0.0:
            return 1, f"explicit zero entry at {at}"
        if r[k] != c[k] and w[k] < 0:
            return 1, f"negative off-diagonal weight at {at}: no CTMC interpretation"
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    order = np.lexsort((hi, lo))
    lo, hi, w = lo[order], hi[order], w[order]
    for k in range(1, len(lo)):
        if lo[k] == lo[k - 1] and hi[k] == hi[k - 1]:
            return 1, f"duplicate entry at ({lo[k]}, {hi[k]})"
    return "ok", (lo, hi, w)


def _csr_from_canonical(n, lo, hi, w):
    diag = np.zeros(n)
    rows = [[] for _ in range(n)]
    for a, b, x in zip(lo, hi, w):
        if a == b:
            diag[a] = x
        else:
            rows[a].append((b, x))
            rows[b].append((a, x))
    rp, col, val = [0], [], []
    for i in range(n):
        for b, x in sorted(rows[i]):
            col.append(b); val.append(x)
        rp.append(len(col))
    return np.array(rp, np.uint64), np.array(col, np.uint32), np.array(val), diag


@pytest.mark.parametrize("name", sorted(CASES))
def test_mm_case_matches_reference_golden(pb, tmp_path, name):
    g = CASES[name]
    path = _write(tmp_path, name, g["body"])
    try:
        e = pb.parse_matrix_market(path)
    except pb.ExpmcError as err:
        assert not g["ok"] and g["kind"] == 2, (name, str(err))
        assert str(err) == g["message"].replace("{path}", path)
        return
    out = _fold_and_check(pb, e, path)
    if g["ok"]:
        assert out[0] == "ok", (name, out)
        rp, col, val, diag = _csr_from_canonical(e.n, *out[1])
        assert e.n == g["n"]
        assert rp.tolist() == g["row_offset"]
        assert col.tolist() == g["neighbor"]
        assert [float(x).hex() for x in val] == g["weight"]
        assert [float(x).hex() for x in diag] == g["diag"]
    else:
        assert out == (g["kind"], g["message"].replace("{path}", path)), name


def _csr_of_golden(pb, g):
    return pb.Csr(g["n"], np.array(g["row_offset"], np.uint64),
                  np.array(g["neighbor"], np.uint32),
                  np.array([float.fromhex(x) for x in g["weight"]]),
                  np.array([float.fromhex(x) for x in g["diag"]]))


@pytest.mark.parametrize("idx", range(len(GOLD["writes"])))
def test_mm_write_is_byte_identical_to_reference(pb, tmp_path, idx):
    g = GOLD["writes"][idx]
    p = tmp_path / "out.mtx"
    pb.write_matrix_market(_csr_of_golden(pb, g), str(p))
    assert p.read_text() == g["text"], g["name"]


def _random_csr(pb, n, m, seed, pattern=False, diag=True):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, n, m)
    b = rng.integers(0, n, m)
    keep = a != b
    lo, hi = np.minimum(a, b)[keep], np.maximum(a, b)[keep]
    key = np.unique(lo.astype(np.int64) * n + hi)
    lo, hi = key // n, key % n
    w = np.ones(len(lo)) if pattern else rng.random(len(lo)) * 10 + 1e-3
    if diag:
        d_idx = rng.choice(n, n // 3, replace=False)
        dw = np.ones(len(d_idx)) if pattern else rng.normal(size=len(d_idx))
        lo = np.concatenate([lo, d_idx]); hi = np.concatenate([hi, d_idx]); w = np.concatenate([w, dw])
    order = np.lexsort((hi, lo))
    rp, col, val, dg = _csr_from_canonical(n, lo[order], hi[order], w[order])
    return pb.Csr(n, rp, col, val, dg), (lo[order], hi[order], w[order])


@pytest.mark.parametrize("pattern", [False, True])
def test_mm_roundtrip_large_parallel_parse(pb, tmp_path, pattern):
    """A file big enough to be split across all host cores (several MiB):
    write -> parse returns the lower-triangle entries in file order."""
    n = 50_000
    csr, (lo, hi, w) = _random_csr(pb, n, 400_000, 3, pattern=pattern)
    p = str(tmp_path / "big.mtx")
    pb.write_matrix_market(csr, p)
    assert os.path.getsize(p) > (3 << 20)
    e = pb.parse_matrix_market(p)
    assert (e.n, e.general, e.pattern) == (n, False, pattern)
    np.testing.assert_array_equal(e.rows, hi.astype(np.uint32))   # lower triangle on disk
    np.testing.assert_array_equal(e.cols, lo.astype(np.uint32))
    np.testing.assert_array_equal(e.weights, w)                   # shortest repr round-trips
    assert e.last_line == 2 + len(w)


def test_mm_error_line_numbers_across_parse_ranges(pb, tmp_path):
    """Errors deep inside a multi-range file report the sequential reader's
    line: the earliest bad line wins, comments/blank lines count."""
    body = ["%%MatrixMarket matrix coordinate real symmetric", "% header comment", "1000 1000 300000"]
    for k in range(300_000):
        if k % 997 == 0:
            body.append("% interleaved comment")
        if k % 1409 == 0:
            body.append("")
        body.append(f"{(k % 999) + 2} 1 {1.0 + k % 7}")
    lines = list(body)
    bad1, bad2 = 250_000, 260_000
    lines[bad2] = "1 1 +2.0"
    lines[bad1] = "1 2000 1.0"
    p = _write(tmp_path, "errs", "\n".join(lines) + "\n")
    with pytest.raises(pb.ExpmcError) as ei:
        pb.parse_matrix_market(p)
    assert str(ei.value) == f"{p}:{bad1 + 1}: index out of range"
    # EOF accounting with a large file
    p2 = _write(tmp_path, "eof", "\n".join(body[:-5]) + "\n% tail\n")
    with pytest.raises(pb.ExpmcError) as ei:
        pb.parse_matrix_market(p2)
    got = 300_000 - 5
    assert str(ei.value) == (f"{p2}:{len(body) - 5 + 2}: unexpected end of file: expected "
                             f"300000 entries, got {got}")


def test_mm_parse_matches_live_reference_on_generated_file(pb, ref, tmp_path):
    """Generated file with comments, CRLF and tabs: parse + (test-side) fold
    equals the live reference's load_matrix_market."""
    rng = np.random.default_rng(7)
    n = 3000
    csr, (lo, hi, w) = _random_csr(pb, n, 20_000, 5)
    out = ["%%MatrixMarket matrix coordinate real general", f"{n} {n} {2 * len(w) - int(np.sum(lo == hi))}"]
    for a, b, x in zip(lo, hi, w):
        out.append(f"{b + 1}\t{a + 1} {float(x)!r}\r")
        if a != b:
            out.append(f"  {a + 1} {b + 1}  {float(x)!r}")
        if rng.random() < 0.01:
            out.append("% c")
    p = _write(tmp_path, "gen", "\n".join(out) + "\n")
    rm = ref.mm_load(p)
    e = pb.parse_matrix_market(p)
    st, (clo, chi, cw) = _fold_and_check(pb, e, p)
    assert st == "ok"
    rp, col, val, dg = _csr_from_canonical(n, clo, chi, cw)
    s = rm.split()
    np.testing.assert_array_equal(rp, s["row_offset"])
    np.testing.assert_array_equal(col, s["neighbor"])
    np.testing.assert_array_equal(val, s["weight"])
    np.testing.assert_array_equal(dg, s["diag"])


def test_mm_writer_matches_live_reference(pb, ref, tmp_path):
    csr, (lo, hi, w) = _random_csr(pb, 2000, 15_000, 9)
    mine, theirs = tmp_path / "m.mtx", tmp_path / "r.mtx"
    pb.write_matrix_market(csr, str(mine))
    ref.mm_write_entries(csr.n, lo, hi, w, str(theirs))
    assert mine.read_bytes() == theirs.read_bytes()


def test_mm_write_errors(pb, tmp_path):
    csr, _ = _random_csr(pb, 10, 20, 1)
    with pytest.raises(pb.ExpmcError, match="cannot open .* for write"):
        pb.write_matrix_market(csr, str(tmp_path / "no" / "such" / "dir.mtx"))


def test_mm_missing_file(pb, tmp_path):
    p = str(tmp_path / "absent.mtx")
    with pytest.raises(pb.ExpmcError, match=f"^cannot open {p}$"):
        pb.parse_matrix_market(p)


# ------------------------------------------------------------ CSR cache (f3)
def test_csr_cache_roundtrip(pb, tmp_path):
    for n, m, diag in [(1, 0, False), (7, 10, True), (5000, 40_000, True)]:
        csr, _ = _random_csr(pb, n, m, n, diag=diag)
        p = str(tmp_path / f"c{n}.csr")
        pb.save_csr(csr, p)
        back = pb.load_csr(p)
        assert back.n == csr.n
        for a in ("row_ptr", "col", "val", "diag"):
            np.testing.assert_array_equal(getattr(back, a), getattr(csr, a))


def test_csr_cache_detects_corruption(pb, tmp_path):
    csr, _ = _random_csr(pb, 300, 2000, 2)
    p = tmp_path / "c.csr"
    pb.save_csr(csr, str(p))
    raw = bytearray(p.read_bytes())
    bad = bytearray(raw)
    bad[len(bad) // 2] ^= 0x10
    (tmp_path / "flip.csr").write_bytes(bytes(bad))
    with pytest.raises(pb.ExpmcError, match="checksum mismatch"):
        pb.load_csr(str(tmp_path / "flip.csr"))
    (tmp_path / "short.csr").write_bytes(bytes(raw[:-8]))
    with pytest.raises(pb.ExpmcError, match="truncated or oversized"):
        pb.load_csr(str(tmp_path / "short.csr"))
    (tmp_path / "magic.csr").write_bytes(b"NOTACSR!" + bytes(raw[8:]))
    with pytest.raises(pb.ExpmcError, match="not an expmc CSR cache file"):
        pb.load_csr(str(tmp_path / "magic.csr"))
    with pytest.raises(pb.ExpmcError, match="cannot open"):
        pb.load_csr(str(tmp_path / "absent.csr"))


def test_build_config_uses_csr_cache(pb, tmp_path, monkeypatch):
    from paper_1904_12759_b200 import inputs

    monkeypatch.setenv("EXPMC_CSR_CACHE", str(tmp_path))
    calls = []
    real = inputs.gen_ws

    def counting(*a):
        calls.append(a)
        return real(*a)

    monkeypatch.setattr(inputs, "gen_ws", counting)
    a = inputs.build_config(3, scale=0.002)
    b = inputs.build_config(3, scale=0.002)
    assert len(calls) == 1 and len(os.listdir(tmp_path)) == 1
    for f in ("row_ptr", "col", "val", "diag"):
        np.testing.assert_array_equal(getattr(a.csr, f), getattr(b.csr, f))
