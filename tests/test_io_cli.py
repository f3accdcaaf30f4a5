"""MPCV1 cost volumes and the CLI `run` driver (
reference proj/src/io.cpp:118-152, proj/tools/mrfmp.cpp:77-166).

CPU: the Python reader / writer round trip and rejections, and the C++
reader's rejections through the CLI (they happen before any device work).
GPU: `mrfmp_cuda run` per method against the reference library's
per-iteration energies on the 4-connected protocol (mrfmp.cpp:91-101).
"""
import os
import subprocess

import numpy as np
import pytest

from paper_1910_10892_b200 import api
from paper_1910_10892_b200 import build as B

CLI = B.CLI_OUT


def _vol(H, W, L, seed):
    return np.random.default_rng(seed).uniform(0.0, 8.0, (H, W, L)).astype(np.float32)


def test_mpcv1_round_trip_and_layout(tmp_path):
    v = _vol(5, 7, 9, 1)
    p = str(tmp_path / "v.mpcv")
    api.save_cost_volume(p, v)
    raw = open(p, "rb").read()
    assert raw[:5] == b"MPCV1" and np.frombuffer(raw[5:17], "<u4").tolist() == [5, 7, 9]
    assert len(raw) == 17 + 4 * v.size
    assert np.array_equal(api.load_cost_volume(p), v)


@pytest.mark.parametrize("mutate,msg", [
    (lambda r: b"MPCV2" + r[5:], "bad magic"),
    (lambda r: r[:12], "truncated header"),
    (lambda r: r[:-4], "truncated payload"),
    (lambda r: r[:5] + np.array([0, 7, 9], "<u4").tobytes() + r[17:], "invalid dimensions"),
    (lambda r: r[:5] + np.array([5, 7, 300], "<u4").tobytes() + r[17:], "invalid dimensions"),
    (lambda r: r[:17] + np.array([np.nan], "<f4").tobytes() + r[21:], "non-finite"),
])
def test_mpcv1_rejections(tmp_path, mutate, msg):
    p = str(tmp_path / "v.mpcv")
    api.save_cost_volume(p, _vol(5, 7, 9, 2))
    bad = str(tmp_path / "bad.mpcv")
    open(bad, "wb").write(mutate(open(p, "rb").read()))
    with pytest.raises(ValueError, match=msg):
        api.load_cost_volume(bad)
    # the C++ reader (mrf/io.hpp) rejects it the same way, before any GPU work
    res = subprocess.run([CLI, "run", "--unary-file", bad, "--out-csv", str(tmp_path / "r.csv"),
                          "--out-labels", str(tmp_path / "l.pgm")], capture_output=True, text=True)
    assert res.returncode == 1 and msg in res.stderr, res.stderr


def test_cli_usage_errors(tmp_path):
    assert subprocess.run([CLI], capture_output=True).returncode == 2
    for args in (["--method", "bogus"], ["--precision", "f64"], ["--iters", "0"], ["--pairwise", "xx"],
                 ["--dirs"], ["--nope", "1"], ["--method", "mf"]):
        res = subprocess.run([CLI, "run", *args, "--out-csv", str(tmp_path / "r.csv")], capture_output=True, text=True)
        assert res.returncode == 2, (args, res.stderr)


def _ref_energies(method, pr, K):
    from oracle import oracle as O

    pr4 = O.Problem(pr.H, pr.W, pr.L, 4, pr.unary, pr.V, pr.w_const, None, 0.5, None)
    if method in ("isgmr", "trwp"):
        labs = [O.forward(method, pr, k, impl="ref", threads=0).labels for k in range(1, K + 1)]
    else:
        labs = [lab for _, lab in O.ref_sgm_iterative(pr, K, "revised" if method == "sgm" else "standard")]
    return [O.ref_energy(pr4, lab) for lab in labs]


@pytest.mark.gpu
@pytest.mark.parametrize("method,dirs,pairwise,trunc", [("isgmr", 4, "tl", 2.0), ("trwp", 8, "tl", 3.0),
                                                        ("sgm", 4, "potts", -1.0), ("sgm-std", 8, "tq", 9.0)])
def test_cli_run_matches_reference(tmp_path, method, dirs, pairwise, trunc):
    import torch

    from oracle import oracle as O
    from paper_1910_10892_b200 import workloads as WL

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not O.have_ref():
        pytest.skip("reference library not present")
    H, W, L, K = 14, 17, 12, 4
    v = WL.stereo_like(H, W, L, 9).reshape(H, W, L)
    vp = str(tmp_path / "u.mpcv")
    api.save_cost_volume(vp, v)
    csv, lab = str(tmp_path / "run.csv"), str(tmp_path / "labels.pgm")
    res = subprocess.run([CLI, "run", "--method", method, "--dirs", str(dirs), "--iters", str(K), "--pairwise", pairwise,
                          "--trunc", str(trunc), "--unary-file", vp, "--weight", "0.75", "--out-csv", csv,
                          "--out-labels", lab], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    rows = [ln.split(",") for ln in open(csv).read().split("\n")[1:] if ln]
    assert [int(r[0]) for r in rows] == list(range(1, K + 1))
    kind = {"potts": WL.potts(L), "tl": WL.truncated_linear(L, trunc), "tq": WL.truncated_quadratic(L, trunc)}[pairwise]
    pr = O.Problem(H, W, L, dirs, v.reshape(-1).copy(), kind, 0.75, None, 0.5, None)
    want = _ref_energies(method, pr, K)
    for r, e in zip(rows, want):
        assert abs(float(r[1]) - e) <= 1e-9 * max(1.0, abs(e)), (r, e)
    assert f"final_energy={float(rows[-1][1]):.10g}" in res.stdout
    raw = open(lab, "rb").read()
    assert raw.startswith(f"P5\n{W} {H}\n65535\n".encode())
    assert len(raw) == len(f"P5\n{W} {H}\n65535\n") + 2 * H * W
