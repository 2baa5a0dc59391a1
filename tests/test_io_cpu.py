"""Data formats and generators either side of the path,
host-only C-ABI entry points, against the reference's own io.cpp /
generators.cpp compiled into oracle/_ref (bit-exact points, byte-equal files,
the same InvalidArgument texts). No GPU needed."""
import os

import numpy as np
import pytest

import paper_2107_06876_b200 as lcn
from oracle.bindings import LcnError, RefLib, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    return RefLib()


def tricky_points(seed=3, n=37, d=5):
    r = np.random.default_rng(seed)
    x = r.standard_normal((n, d)) * 10.0 ** r.integers(-12, 12, (n, d))
    x[0, 0], x[1, 1], x[2, 2] = 0.1, -0.0, 1.0 / 3.0
    return x


@pytest.mark.parametrize("binary", [True, False])
def test_points_files_match_reference(ref, tmp_path, binary):
    x = tricky_points()
    ours, theirs = str(tmp_path / "ours.pts"), str(tmp_path / "theirs.pts")
    lcn.write_points_file(ours, x, binary)
    ref.points_write(theirs, x, binary)
    assert open(ours, "rb").read() == open(theirs, "rb").read()  # byte-equal files
    for path in (ours, theirs):
        a, b = lcn.read_points_file(path), ref.points_read(path)
        assert a.shape == x.shape
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
        assert np.array_equal(a.view(np.uint64), x.view(np.uint64))  # 17 digits round-trip exactly


def test_text_comments_and_blank_lines(ref, tmp_path):
    path = str(tmp_path / "c.txt")
    with open(path, "w") as f:
        f.write("# header comment\n\n  2 3\n1 2 3\n   # row comment\n\t\n4.5 -6e-3 7\n")
    a = lcn.read_points_file(path)
    assert np.array_equal(a, ref.points_read(path))
    assert np.array_equal(a, [[1, 2, 3], [4.5, -6e-3, 7]])


@pytest.mark.parametrize("content,binary", [
    (b"", False),
    (b"0 3\n", False),
    (b"2 2\n1 2\n", False),
    (b"2 2\n1 2\n3\n", False),
    (b"1 2\n1 nan\n", False),
    (b"LCNPTS1" + (2).to_bytes(8, "little") + (2).to_bytes(8, "little") + b"\0" * 16, True),
    (b"LCNPTS1" + (0).to_bytes(8, "little") + (2).to_bytes(8, "little"), True),
    (b"LCNPTS1" + (1).to_bytes(8, "little") + (1).to_bytes(8, "little") + np.array([np.inf]).tobytes(), True),
])
def test_malformed_files_raise_reference_errors(ref, tmp_path, content, binary):
    path = str(tmp_path / "bad.pts")
    with open(path, "wb") as f:
        f.write(content)
    with pytest.raises(LcnError) as theirs:
        ref.points_read(path)
    with pytest.raises(lcn.InvalidArgument) as ours:
        lcn.read_points_file(path)
    assert theirs.value.kind == "InvalidArgument" and str(ours.value) == theirs.value.msg


def test_missing_file(ref, tmp_path):
    path = str(tmp_path / "nope.pts")
    with pytest.raises(lcn.InvalidArgument, match="cannot open point file"):
        lcn.read_points_file(path)
    with pytest.raises(LcnError):
        ref.points_read(path)


@pytest.mark.parametrize("n,d,seed", [(1, 1, 0), (200, 3, 7), (64, 40, 2 ** 63 + 5)])
def test_uniform_ball_bit_exact(ref, n, d, seed):
    a = lcn.sample_uniform_ball(n, d, seed)
    assert np.array_equal(a.view(np.uint64), ref.sample_uniform_ball(n, d, seed).view(np.uint64))
    assert np.all(np.linalg.norm(a, axis=1) <= 1.0 + 1e-12)


@pytest.mark.parametrize("n,d,c,D,r,seed", [(100, 2, 4, 10.0, 0.5, 1), (300, 16, 9, 3.0, 1.5, 42),
                                            (5, 1, 1, 1.0, 0.0, 3)])
def test_clustered_bit_exact(ref, n, d, c, D, r, seed):
    p, q, ctr = lcn.sample_clustered(n, d, c, D, r, seed)
    rp, rq, rc = ref.sample_clustered(n, d, c, D, r, seed)
    for a, b in ((p, rp), (q, rq), (ctr, rc)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_generator_errors(ref):
    with pytest.raises(lcn.InvalidArgument, match="sample_uniform_ball: n and d must be positive"):
        lcn.sample_uniform_ball(0, 3, 1)
    with pytest.raises(lcn.InvalidArgument, match="D must be positive"):
        lcn.sample_clustered(4, 2, 2, -1.0, 0.5, 1)
    with pytest.raises(lcn.InvalidArgument, match="sizes must be positive") as ours:
        lcn.sample_clustered(4, 2, 0, 1.0, 0.5, 1)
    with pytest.raises(LcnError) as theirs:
        ref.sample_clustered(4, 2, 0, 1.0, 0.5, 1)
    assert str(ours.value) == theirs.value.msg


def test_runner_host_logic():
    """config_from_json / config_to_json round trip, mix_seed (runner.cpp:175-180)
    against the configs.py mirror, lsh_bucket_count (runner.cpp:206-216)."""
    from paper_2107_06876_b200 import configs, runner
    j = {"problem": {"generator": "clustered", "n": 10, "d": 2, "c": 3, "D": 4.0, "r": 0.5},
         "variants": ["lcn"], "lsh": {"scheme": "cross-polytope", "rows-per-band": 2}, "seeds": [4, 9]}
    c = runner.config_from_json(j)
    assert runner.config_from_json(runner.config_to_json(c)) == c
    for s in (0, 1, 2 ** 64 - 1):
        for salt in (1, 2, 3, 4):
            assert runner.mix_seed(s, salt) == configs.mix_seed(s, salt)
    assert runner.lsh_bucket_count(c, 1000, 800, 20) == 6  # llround(sqrt(800 / 20)), already even
    assert runner.lsh_bucket_count(c, 1000, 1000, 20) == 8  # llround(sqrt(50)) = 7 -> even for cross-polytope
    with pytest.raises(lcn.InvalidArgument, match="unknown problem generator"):
        runner.config_from_json({"problem": {"generator": "x"}})
