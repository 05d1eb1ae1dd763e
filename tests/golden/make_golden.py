#!/usr/bin/env python
"""Regenerate the golden fixtures under tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libexpmc_ref.so, compiled from /root/reference by
`make -C oracle`) and from curand's Philox (compiled host-side with nvcc).

The reference ships no tests or fixtures (tests/ is absent), so
these are produced from the compiled reference itself:
  rng.json      RngStream sequences / exp_time draws     rng.hpp:14-63, sampler.cpp:10-16
  split.json    split() of small matrices                 sparse_matrix.cpp:101-142
  estimates.json entry/vector/tc estimates, workers = 1   estimator.cpp:169-318
  advance.json  advance() end states / jumps per stream   sampler.cpp:36-49
  ba.json       generate({ScaleFree, ...}) CSR            generators.cpp:58-103
  philox.json   Philox4x32-10 known answers (curand)
  mm.json       load/write_matrix_market outcomes       matrix_market.cpp:51-207

usage: python tests/golden/make_golden.py [mm]   (needs /root/reference + nvcc)
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

ref = oracle.Ref()


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=0, sort_keys=True)
        f.write("\n")


def fl(a):
    """float64 array -> list of hex strings (bit-exact round trip)."""
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64)]


def csr_of(rm):
    s = rm.split()
    return s


def small_matrices():
    """name -> (n, rows, cols, weights) entry lists fed to from_entries."""
    mats = {}
    mats["p3"] = (3, [0, 1, 1], [1, 2, 1], [1.0, 3.0, 0.5])
    mats["single_edge"] = (2, [0], [1], [1.0])
    mats["empty3"] = (3, [], [], [])
    mats["star5"] = (5, [0, 0, 0, 0], [1, 2, 3, 4], [1.0, 1.0, 1.0, 1.0])
    # weighted path with diagonal and a mirrored (lower-triangle) entry
    mats["wpath6"] = (6, [0, 2, 2, 4, 5, 3, 0], [1, 1, 3, 3, 4, 3, 0],
                      [0.5, 2.0, 1.5, 4.0, 0.25, -1.0, 2.0])
    # 4x4 FD Laplacian (diag -4, off +1)
    r, c, w = [], [], []
    L = 4
    for i in range(L * L):
        x, y = i % L, i // L
        r.append(i); c.append(i); w.append(-4.0)
        if x + 1 < L:
            r.append(i); c.append(i + 1); w.append(1.0)
        if y + 1 < L:
            r.append(i); c.append(i + L); w.append(1.0)
    mats["fd2d_4"] = (L * L, r, c, w)
    rng = np.random.default_rng(11)
    r, c, w = [], [], []
    for _ in range(60):
        i, j = rng.integers(0, 25, 2)
        if i < j and (i, j) not in zip(r, c):
            r.append(int(i)); c.append(int(j)); w.append(float(rng.integers(1, 9)) / 4.0)
    for i in range(25):
        r.append(i); c.append(i); w.append(float(rng.normal()))
    mats["rand25_weighted"] = (25, r, c, w)
    return mats


def main():
    # ---------------------------------------------------------------- rng
    rng = {
        "pcg32_demo_42_54_u32": [int(x) for x in ref.rng_draws(42, 54, 0, 8)],
        "s1_0": {
            "u32": [int(x) for x in ref.rng_draws(1, 0, 0, 6)],
            "u64": [str(int(x)) for x in ref.rng_draws(1, 0, 1, 6)],
            "uniform": fl(ref.rng_draws(1, 0, 2, 6)),
            "uniform_pos": fl(ref.rng_draws(1, 0, 3, 6)),
            "uniform_index_10": [int(x) for x in ref.rng_draws(1, 0, 4, 6, 10)],
        },
        "s7_3_uniform": fl(ref.rng_draws(7, 3, 2, 6)),
        "s2024_99_uniform_index_1000": [int(x) for x in ref.rng_draws(2024, 99, 4, 6, 1000)],
        "exp_time_1_0_rate2": fl(ref.exp_times(1, 0, 2.0, 6)),
        "exp_time_5_8_rate0_5": fl(ref.exp_times(5, 8, 0.5, 6)),
    }
    dump("rng.json", rng)

    # -------------------------------------------------- split / estimates
    mats = small_matrices()
    split_out, est_out, adv_out = {}, {}, {}
    for name, (n, r, c, w) in mats.items():
        rm = ref.matrix_from_entries(n, r, c, w)
        s = rm.split()
        split_out[name] = {
            "n": n, "entries": [r, c, fl(w)],
            "row_offset": [int(x) for x in s["row_offset"]],
            "neighbor": [int(x) for x in s["neighbor"]],
            "weight": fl(s["weight"]), "diag": fl(s["diag"]), "d": fl(s["d"]),
            "rate": fl(s["rate"]), "cum": fl(s["cum"]),
            "uniform_row": [int(x) for x in s["uniform_row"]],
            "dbar": float(s["dbar"]).hex(), "dmax": int(s["dmax"]),
        }
        v = np.array([((k * 7) % 5) / 2.0 - 0.5 for k in range(n)])
        vpos = np.abs(v) + 0.25
        cases = []
        for split_mode in (0, 1):
            for i in sorted(set([0, n // 2, n - 1])):
                if n == 0:
                    continue
                val, se, j = rm.entry_estimate(v, i, 0.8, 8, 3000, split_mode, 31, workers=1)
                cases.append({"kind": "entry", "i": i, "splitting": split_mode, "beta": 0.8,
                              "n_steps": 8, "samples": 3000, "seed": 31, "value": val.hex(),
                              "se": se.hex(), "jumps": j})
            if n:
                vals, se, j, vs = rm.vector_estimate(vpos, 0.8, 8, 4000, split_mode, 32, workers=1)
                cases.append({"kind": "vector", "splitting": split_mode, "beta": 0.8,
                              "n_steps": 8, "samples": 4000, "seed": 32, "values": fl(vals),
                              "se": se.hex(), "jumps": j, "v_sum": vs.hex()})
                val, se, j = rm.tc_estimate(0.8, 8, 4000, split_mode, 33, workers=1)
                cases.append({"kind": "tc", "splitting": split_mode, "beta": 0.8, "n_steps": 8,
                              "samples": 4000, "seed": 33, "value": val.hex(), "se": se.hex(),
                              "jumps": j})
        est_out[name] = {"v": fl(v), "vpos": fl(vpos), "cases": cases}
        if n and int(s["row_offset"][-1]) > 0:
            start = int(np.argmax(np.diff(s["row_offset"])))
            end, jumps = rm.advance_many(77, start, 0.5, 64)
            adv_out[name] = {"start": start, "dt": 0.5, "seed": 77,
                             "end": [int(x) for x in end], "jumps": [int(x) for x in jumps]}
    dump("split.json", split_out)
    dump("estimates.json", est_out)
    dump("advance.json", adv_out)

    # --------------------------------------------------------------- BA
    ba = {}
    for n, m0, seed in ((300, 4, 9), (1000, 5, 1)):
        s = ref.generate(1, n, m0=m0, seed=seed).split()
        ba[f"n{n}_m{m0}_s{seed}"] = {"n": n, "m0": m0, "seed": seed,
                                     "row_offset": [int(x) for x in s["row_offset"]],
                                     "neighbor": [int(x) for x in s["neighbor"]]}
    dump("ba.json", ba)

    # ---------------------------------------------------- Philox (curand)
    src = r'''
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
int main() {
  unsigned c[][6] = {{0,0,0,0,0,0},
    {0xffffffffu,0xffffffffu,0xffffffffu,0xffffffffu,0xffffffffu,0xffffffffu},
    {0x243f6a88u,0x85a308d3u,0x13198a2eu,0x03707344u,0xa4093822u,0x299f31d0u},
    {7,1,2,0x454e5452u,3,0},{0xffffffffu,5,123,0x454e5452u,42,0}};
  for (auto& k : c) {
    uint4 r = curand_Philox4x32_10(make_uint4(k[0],k[1],k[2],k[3]), make_uint2(k[4],k[5]));
    printf("%u %u %u %u %u %u %u %u %u %u\n",k[0],k[1],k[2],k[3],k[4],k[5],r.x,r.y,r.z,r.w);
  }
}
'''
    with tempfile.TemporaryDirectory() as d:
        with open(os.path.join(d, "k.cu"), "w") as f:
            f.write(src)
        subprocess.run(["nvcc", "-o", os.path.join(d, "k"), os.path.join(d, "k.cu")],
                       check=True, capture_output=True)
        out = subprocess.run([os.path.join(d, "k")], check=True, capture_output=True,
                             text=True).stdout
    kat = [[int(x) for x in ln.split()] for ln in out.strip().splitlines()]
    dump("philox.json", {"source": "curand_Philox4x32_10 (CUDA 12.9), host build",
                         "cases": [{"ctr": k[:4], "key": k[4:6], "out": k[6:]} for k in kat]})
    print("golden fixtures written to", HERE)


def mm_goldens():
    """mm.json: load_matrix_market outcomes for tests/mm_cases.py and
    write_matrix_market texts, from the reference (matrix_market.cpp)."""
    sys.path.insert(0, os.path.dirname(HERE))
    from mm_cases import CASES

    def csr_json(rm):
        s = rm.split()
        return {"n": rm.n, "row_offset": [int(x) for x in s["row_offset"]],
                "neighbor": [int(x) for x in s["neighbor"]], "weight": fl(s["weight"]),
                "diag": fl(s["diag"])}

    cases, writes = [], []
    with tempfile.TemporaryDirectory() as d:
        for name, body in CASES:
            p = os.path.join(d, name + ".mtx")
            with open(p, "w", newline="") as f:
                f.write(body)
            try:
                out = {"ok": True, **csr_json(ref.mm_load(p))}
            except oracle.RefError as e:
                out = {"ok": False, "kind": e.kind, "message": str(e).replace(p, "{path}")}
            cases.append({"name": name, "body": body, **out})
        mats = small_matrices()
        mats["awkward_reals"] = (6, [0, 0, 1, 2, 3, 4, 5], [1, 2, 3, 4, 5, 5, 0],
                                 [0.1, 1.0 / 3.0, 1e-300, 1e300, 5e-324, 123456789.125, 7.0])
        for name, (n, r, c, w) in sorted(mats.items()):
            rm = ref.matrix_from_entries(n, r, c, w)
            p = os.path.join(d, name + ".out.mtx")
            ref.mm_write_entries(n, r, c, w, p)
            with open(p) as f:
                writes.append({"name": name, **csr_json(rm), "text": f.read()})
    dump("mm.json", {"source": "reference load/write_matrix_market (oracle/_ref)",
                     "cases": cases, "writes": writes})


if __name__ == "__main__":
    if sys.argv[1:] == ["mm"]:
        mm_goldens()
    else:
        main()
        mm_goldens()
