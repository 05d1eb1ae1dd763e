"""CPU tests of the host side: C-ABI exports, host validation, the input
generators (BA restated draw-for-draw from the reference), parameter
handling, the row-shard planner and the multi-rank gather (gloo,
world_size 2), and the reference arm of bench.py.  No GPU needed."""
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_header_symbol(pb):
    hdr = open(os.path.join(ROOT, "include", "expmc_b200.h")).read()
    names = sorted(set(re.findall(r"\b(expmc_(?:cuda|gen|csr|mm)_\w+)\s*\(", hdr)))
    assert len(names) >= 25
    L = pb.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding declares exactly these
    from paper_1904_12759_b200._lib import SIGNATURES

    assert sorted(n for n, _, _ in SIGNATURES) == names
    assert L.expmc_cuda_abi_version() == 1


def test_host_validation_before_device(pb):
    with pytest.raises(ValueError, match=r"row_ptr\[0\] must be 0"):
        pb.SplitMatrix.from_csr(2, np.array([1, 1, 2], np.uint64), np.array([1, 0], np.uint32),
                                np.ones(2))
    with pytest.raises(ValueError, match="row_ptr must be non-decreasing"):
        pb.SplitMatrix.from_csr(2, np.array([0, 2, 1], np.uint64), np.array([1, 0], np.uint32),
                                np.ones(2))
    with pytest.raises(ValueError, match=r"non-finite weight at \(1, 1\)"):
        pb.SplitMatrix.from_csr(2, np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32),
                                np.ones(2), np.array([0.0, np.inf]))


def test_path_params_mirror_reference(pb):
    P = pb.PathParams
    with pytest.raises(ValueError, match="beta must be positive and finite"):
        P(beta=float("nan")).validate()
    with pytest.raises(ValueError, match="n_steps must be >= 1"):
        P(n_steps=0).validate()
    with pytest.raises(ValueError, match="samples must be >= 1"):
        P(samples=0).validate()
    with pytest.raises(ValueError, match="beta and dt must be positive"):
        P.with_dt(1.0, 0.0, 10, pb.Splitting.Strang, 0)
    # llround semantics (estimator.cpp:156-157): half away from zero, >= 1
    assert P.with_dt(1.0, 0.4, 10, pb.Splitting.Strang, 0).n_steps == 3  # 2.5 -> 3
    assert P.with_dt(1.0, 10.0, 10, pb.Splitting.Strang, 0).n_steps == 1
    assert P.with_dt(1.0, 0.03125, 10, pb.Splitting.Lie, 0).n_steps == 32
    p = P(beta=2.0, n_steps=8)
    assert p.dt() == 0.25
    d = P()  # estimator.hpp:16-33 defaults
    assert (d.beta, d.n_steps, d.samples, d.splitting, d.seed) == (1.0, 32, 1_000_000,
                                                                    pb.Splitting.Strang, 0)


def test_ba_generator_matches_reference_golden(pb):
    g = json.load(open(os.path.join(GOLD, "ba.json")))
    for k, c in g.items():
        csr = pb.gen_ba(c["n"], c["m0"], c["seed"])
        assert list(csr.row_ptr) == c["row_offset"], k
        assert list(csr.col) == c["neighbor"], k
        assert np.all(csr.val == 1.0) and np.all(csr.diag == 0.0)


def test_ba_generator_matches_reference_directly(pb, ref):
    csr = pb.gen_ba(20_000, 8, 1)
    s = ref.generate(1, 20_000, m0=8, seed=1).split()
    assert np.array_equal(csr.row_ptr, s["row_offset"])
    assert np.array_equal(csr.col, s["neighbor"])


def _check_symmetric(csr):
    rp = csr.row_ptr.astype(np.int64)
    rows = np.repeat(np.arange(csr.n), np.diff(rp))
    a = set(zip(rows.tolist(), csr.col.tolist()))
    assert all((j, i) in a for i, j in a)
    assert all(i != j for i, j in a)
    for i in range(csr.n):
        seg = csr.col[rp[i]:rp[i + 1]]
        assert np.all(np.diff(seg.astype(np.int64)) > 0)


def test_fd_generators(pb):
    c2 = pb.gen_fd(2, 5, 1.0)
    assert c2.n == 25 and c2.nnz == 2 * 2 * 5 * 4
    assert np.all(c2.diag == -4.0) and np.all(c2.val == 1.0)
    _check_symmetric(c2)
    h = 1.0 / 257.0
    assert 1.0 / (h * h) == 66049.0  # config 4 scale is exact in fp64
    c3 = pb.gen_fd(3, 4, 25.0)
    assert c3.n == 64 and c3.nnz == 3 * 2 * 4 * 4 * 3
    assert np.all(c3.diag == -6.0 * 25.0)
    _check_symmetric(c3)


def test_ws_generator(pb):
    c = pb.gen_ws(2000, 5, 0.1, 1)
    assert c.nnz == 2 * 2000 * 5  # rewiring keeps the edge count
    _check_symmetric(c)
    c2 = pb.gen_ws(2000, 5, 0.1, 1)
    assert np.array_equal(c.col, c2.col)  # deterministic
    ring = pb.gen_ws(100, 2, 0.0, 1)
    assert np.all(np.diff(ring.row_ptr.astype(np.int64)) == 4)


def test_vectors_and_row_sample(pb, orc):
    v = pb.gen_vector(0, 1000, 2)
    assert np.array_equal(v, orc.rng_draws(2, 0, 2, 1000))  # RngStream(2,0).uniform()
    v1 = pb.gen_vector(1, 1000, 2)
    assert np.allclose(v1, 2 * v - 1) and v1.min() >= -1 and v1.max() < 1
    b = pb.gen_vector(2, 512, 2, side=8, sigma=0.1)
    assert b.max() < 2.0 and b.min() >= 0.0
    rs = pb.gen_row_sample(10_000, 500, 4)
    assert len(np.unique(rs)) == 500 and np.all(np.diff(rs.astype(np.int64)) > 0)


def test_n_rule(pb):
    assert pb.n_rule(1.0, np.array([0.0, -1.0, -2.0])) == 32
    assert pb.n_rule(0.02, np.array([15729.0])) == 512  # config 5
    assert pb.n_rule(1e-4, np.array([3 * 66049.0])) == 32  # config 4
    assert pb.n_rule(1.0, np.array([40.0])) == 64


def test_shard_planner():
    from paper_1904_12759_b200.shard import plan_shards

    for n, w in ((10, 3), (7, 8), (10_000_000, 8), (0, 2)):
        p = plan_shards(n, w)
        assert p[0][0] == 0 and p[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(p, p[1:]))
        sizes = [hi - lo for lo, hi in p]
        assert max(sizes) - min(sizes) <= 1


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import oracle
    import paper_1904_12759_b200 as pb
    from paper_1904_12759_b200.shard import gather_slices, shard_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Oracle()
    csr = pb.gen_ba(600, 3, 7)
    s = o.split(csr)
    v = pb.gen_vector(1, csr.n, 2)
    rows = np.arange(csr.n, dtype=np.uint32)
    mine = shard_rows(rows, rank, world)
    # CPU model of the walker stands in for the GPU kernel on this rank
    val, se, j = o.fast_entries(s, v, mine, 0.2, 32, 1000, 1, 5, 32)
    gv, gs, gj = gather_slices(torch.from_numpy(val), torch.from_numpy(se),
                               torch.from_numpy(j.astype(np.int64)), len(rows))
    if rank == 0:
        q.put((gv.numpy().copy(), gs.numpy().copy(), gj.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_multi_rank_gather_gloo_is_bitwise_g_invariant(orc):
    import torch.multiprocessing as mp

    import paper_1904_12759_b200 as pb

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gv, gs, gj = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    csr = pb.gen_ba(600, 3, 7)
    s = orc.split(csr)
    v = pb.gen_vector(1, csr.n, 2)
    val, se, j = orc.fast_entries(s, v, np.arange(csr.n, dtype=np.uint32), 0.2, 32, 1000, 1, 5,
                                  32)
    assert np.array_equal(gv, val) and np.array_equal(gs, se)
    assert np.array_equal(gj, j.astype(np.int64))


def _fake_vector_shard(n, M):
    """Deterministic stand-in for one rank's vector_estimate_rows (the CUDA
    kernel cannot run here): depends only on the shard's row range."""
    def fn(lo, hi):
        r = np.random.default_rng(1000 + lo)
        vals = r.uniform(size=n) / M
        return vals, float(vals.sum() * M), float((vals ** 2).sum() * M * M), 2 ** 40 + 3 * lo + hi
    return fn


def _gloo_vec_worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_1904_12759_b200.estimator import PathParams
    from paper_1904_12759_b200.shard import tc_estimate_sharded, vector_estimate_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, M = 97, 5000
    v = np.linspace(0.5, 2.0, n)
    p = PathParams(0.3, 16, M, seed=4)
    fake = _fake_vector_shard(n, M)
    ve = vector_estimate_sharded(None, v, p, shard_fn=fake)
    te = tc_estimate_sharded(None, p, n, shard_fn=lambda lo, hi: fake(lo, hi)[1:])
    if rank == 0:
        q.put((ve.values.copy(), ve.std_error_global, ve.total_jumps, ve.v_sum, te))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_vector_and_tc_shards_combine_in_rank_order_gloo(world):
    """Theorem-2 start-row shards over gloo ranks: per-end vectors and
    tallies gathered and added in rank order, jumps (u64) carried exactly."""
    import torch.multiprocessing as mp

    from paper_1904_12759_b200.shard import combine_tc_shards, combine_vector_shards, plan_shards

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world * 7 + os.getpid() % 500
    procs = [ctx.Process(target=_gloo_vec_worker, args=(r, world, port, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    vals, se, jm, vs, te = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    n, M = 97, 5000
    fake = _fake_vector_shard(n, M)
    parts = [fake(lo, hi) for lo, hi in plan_shards(n, world)]
    want = combine_vector_shards(parts, M, float(np.linspace(0.5, 2.0, n).sum()))
    assert np.array_equal(vals, want.values) and se == want.std_error_global
    assert jm == want.total_jumps == sum(p[3] for p in parts) and vs == want.v_sum
    wt = combine_tc_shards([p[1:] for p in parts], M)
    assert te == wt


_REF_ARM_CHILD = r"""
import json, runpy, sys
sys.argv = ["bench.py"] + sys.argv[1:]
try:
    runpy.run_path(%r, run_name="__main__")
except SystemExit as e:
    assert not e.code, e.code
maps = open("/proc/self/maps").read()
print(json.dumps({"maps_product": "libexpmc_b200" in maps, "maps_ref": "libexpmc_ref" in maps,
                  "product_imported": "paper_1904_12759_b200" in sys.modules}))
"""


@pytest.mark.parametrize("cfg,scale", [(1, 0.05), (2, 0.02), (4, 0.0005)])
def test_bench_reference_arm_cpu(ref, pb, cfg, scale):
    """--impl reference runs the reference without the product library in
    its process, and prints the same config dict as the GPU arm."""
    code = _REF_ARM_CHILD % os.path.join(ROOT, "bench.py")
    out = subprocess.run([sys.executable, "-c", code, "--impl", "reference",
                          "--config", str(cfg), "--scale", str(scale), "--steps", "1",
                          "--warmup", "0", "--cpu-seconds", "0.3"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.strip().splitlines() if x.startswith("{")]
    line, maps = lines[-2], lines[-1]
    assert maps == {"maps_product": False, "maps_ref": True, "product_imported": False}
    assert line["impl"] == "reference" and line["value"] > 0
    for k in ("metric", "unit", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert k in line
    cb = line["cpu_baseline"]
    # path-only rate: a few rows at samples = F W minus the same rows at
    # samples = 1 (None when the walkers stay below the timing noise)
    assert cb["kind"] == "reference" and "path_only_how" in cb
    assert cb["path_only_value"] is None or cb["path_only_value"] > 0
    assert 0.0 <= cb["setup_share"] <= 1.0 and cb["setup_per_call_s"] > 0
    sys.path.insert(0, ROOT)
    import bench

    c = pb.build_config(cfg, scale, lambda_max=(ref.generate(1, max(1000, int(1e5 * scale)), m0=5,
                                                             seed=1).lambda_max(100)
                                                if cfg == 2 else None))
    rows = c.csr.n if c.rows is None else len(c.rows)
    want = bench.config_dict(c.idx, c.name, c.csr.n, c.csr.nnz, rows, c.walkers, c.n_steps,
                             c.beta, 1)
    assert line["config"] == want


def _build_cpp_demo(out_dir):
    exe = os.path.join(str(out_dir), "api_demo")
    lib_dir = os.path.join(ROOT, "paper_1904_12759_b200")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "api_demo.cpp"), "-L", lib_dir, "-lexpmc_b200",
           f"-Wl,-rpath,{lib_dir}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_header_api_compiles_and_links(tmp_path, pb):
    _build_cpp_demo(tmp_path)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"),
                    reason="reference headers not present (GPU box)")
def test_integration_binding_compiles_against_reference(tmp_path):
    """The C++ binding INTEGRATION.md asks a maintainer to add next to
    proj/include/expmc/estimator.hpp compiles against the reference's own
    headers and include/expmc_b200.h (syntax and types only)."""
    import shutil
    import subprocess

    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    doc = open(os.path.join(root, "INTEGRATION.md")).read()
    i = doc.index("// proj/include/expmc/gpu_backend.hpp")
    src = tmp_path / "gpu_backend.cpp"
    src.write_text(doc[i:doc.index("```", i)] + "\nint main() { return 0; }\n")
    r = subprocess.run([gxx, "-std=c++20", "-fsyntax-only", "-Wno-pragma-once-outside-header",
                        "-I/root/reference/proj/include", "-I" + os.path.join(root, "include"),
                        str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_bench_roofline_levels_and_evidence():
    """bench.make_roofline: config 5 is judged against the measured HBM peak,
    the cache-resident configs against the measured L2 gather ceiling
    (profiles/r02/l2_gather_peak.json); DRAM traffic, sector efficiency and the
    same-source flag come from the committed ncu captures; the §8d byte model
    and the design-byte fraction are both present."""
    import types

    sys.path.insert(0, ROOT)
    import bench

    l2 = bench._load_json("profiles", "r02", "l2_gather_peak.json")
    assert l2 and l2["gbs_model_64B"] > 6000 and "how" in l2
    for idx, bound in ((5, "hbm"), (4, "l2"), (1, "l2")):
        prof = bench._load_json("profiles", "r02", f"ncu_cfg{idx}.json")
        assert prof and prof["dram_bytes_per_launch"] > 0 and prof["source_sha"]
        jumps, entries, ms = 3.2e9, 1e7, 44.0
        r = bench.make_roofline(types.SimpleNamespace(idx=idx), jumps, entries, ms, 1.0)
        assert r["bound"] == bound and r["unit"] == "GB/s"
        balg = 64.0 * jumps + 48.0 * entries
        assert r["algorithmic_bytes_per_launch"] == balg
        assert abs(r["achieved"] - balg / (ms / 1e3) / 1e9) < 1e-6 * r["achieved"]
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
        assert r["design_bytes_per_launch"] == 32.0 * jumps + 48.0 * entries
        assert r["traffic"] == prof["dram_bytes_per_launch"]
        assert r["traffic_same_source"] == (prof["source_sha"] == bench.source_sha())
        assert "sector_efficiency" in r and "frac_dram_measured" in r
    # reduced-scale runs do not borrow the full-size capture
    r = bench.make_roofline(types.SimpleNamespace(idx=5), 1e6, 1e4, 1.0, 0.01)
    assert r["traffic"] is None
