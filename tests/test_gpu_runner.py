"""The runner over the GPU path against the
reference's own run_all (runner.cpp:344-418, compiled into oracle/_ref) on the
same JSON configs: per (variant, seed) record the same keys, sizes, budgets,
iteration counts, error texts, and distance / rel-err-d / PCC / IoU within the
fp64-storage bar."""
import json
import os

import numpy as np
import pytest

import paper_2107_06876_b200 as lcn
from paper_2107_06876_b200 import runner

pytestmark = pytest.mark.gpu

CONFIGS = [
    {"problem": {"generator": "clustered", "n": 240, "d": 4, "c": 4, "D": 8.0, "r": 1.0},
     "variants": ["full", "sparse", "lcn", "nystrom"], "lambda": 0.5, "budget": {"neighbors": 30, "landmarks": 12},
     "max-iters": 300, "seeds": [1, 2], "strict-deterministic": True},
    {"problem": {"generator": "uniform-ball", "n": 300, "m": 260, "d": 6},
     "variants": ["full", "lcn", "sparse"], "lambda": 0.2, "heads": 3,
     "lsh": {"scheme": "cross-polytope", "bands": 2}, "budget": {"neighbors": 25, "landmarks": 16},
     "max-iters": 200, "seeds": [7], "strict-deterministic": True},
    {"problem": {"generator": "uniform-ball", "n": 500, "d": 3}, "variants": ["lcn", "nystrom", "bogus"],
     "lambda": 0.1, "landmark-method": "kmeans++-sampling", "lsh": {"bands": 2, "buckets-per-fn": 6},
     "tol": 0.0, "max-iters": 40, "seeds": [3], "strict-deterministic": True},
]


def compare(ours, theirs):
    assert [(r["variant"], r["seed"]) for r in ours] == [(r["variant"], r["seed"]) for r in theirs]
    for a, b in zip(ours, theirs):
        assert set(a) == set(b), (a, b)
        for k in ("n", "m", "budget", "iters", "converged"):
            assert a[k] == b[k], (k, a, b)
        assert a.get("error") == b.get("error")
        for k in ("distance", "rel-err-d", "pcc", "iou", "marginal-err"):
            if k in b:
                assert abs(a[k] - b[k]) <= 1e-6 * max(1.0, abs(b[k])), (k, a[k], b[k])
        if "head-distances" in b:
            assert np.allclose(a["head-distances"], b["head-distances"], rtol=1e-8, atol=0)


@pytest.mark.parametrize("k", range(len(CONFIGS)))
def test_runner_matches_reference(ref, k):
    cfg = CONFIGS[k]
    ctx = lcn.Context(0, store_fp64=True)
    ours = runner.run_all(runner.config_from_json(cfg), ctx)
    compare(ours, ref.run_all_json(cfg))


def test_runner_files_and_outputs(ref, tmp_path):
    p = lcn.sample_uniform_ball(120, 5, 11)
    q = lcn.sample_uniform_ball(90, 5, 12) * 0.7
    pp, qq = str(tmp_path / "p.pts"), str(tmp_path / "q.txt")
    lcn.write_points_file(pp, p, True)
    lcn.write_points_file(qq, q, False)
    cfg = {"problem": {"generator": "file", "p": pp, "q": qq}, "variants": ["full", "sparse", "lcn"],
           "lambda": 0.3, "budget": {"neighbors": 15, "landmarks": 10}, "seeds": [5],
           "strict-deterministic": True, "output": str(tmp_path / "out.csv")}
    ctx = lcn.Context(0, store_fp64=True)
    c = runner.config_from_json(cfg)
    recs = runner.run_all(c, ctx)
    compare(recs, ref.run_all_json(cfg))
    code = runner.write_outputs(c, recs, str(tmp_path / "out.json"))
    lines = open(cfg["output"]).read().splitlines()
    assert lines[0] == runner.CSV_HEADER
    assert len(lines) == 1 + sum("error" not in r for r in recs)
    j = json.load(open(tmp_path / "out.json"))
    assert j["config"] == runner.config_to_json(c) and j["records"] == recs
    assert code == (2 if any("error" in r for r in recs) else 0)


def test_runner_bp_matches_reference(ref):
    cfg = {"problem": {"generator": "clustered", "n": 120, "d": 3, "c": 3, "D": 6.0, "r": 1.0},
           "variants": ["full", "sparse", "lcn", "nystrom"], "lambda": 0.4, "bp": {"enabled": True, "deletion-cost": 2.5},
           "budget": {"neighbors": 20, "landmarks": 10}, "max-iters": 150, "seeds": [4], "strict-deterministic": True}
    ours = runner.run_all(runner.config_from_json(cfg), lcn.Context(0, store_fp64=True))
    compare(ours, ref.run_all_json(cfg))
