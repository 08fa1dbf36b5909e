"""Oracle pins from the worked examples under tests/golden/.

Each fixture is a small text file: '#' lines give the citation (PAPER.md P:line or
SPEC.md S:line and the passage), the rest are 'key: value' lines.  Values are the
paper's / SPEC's hand traces, never outputs of the CUDA path.  Lists are space
separated; ';' separates rows; '|' separates the fields of one 'case:' line.
"""
import glob
import os

import numpy as np
import pytest

import synth
from oracle import oracle as O
from oracle import theory as TH

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FILES = sorted(glob.glob(os.path.join(GOLDEN, "*.txt")))


def parse(path):
    fx = {"case": []}
    cite = [ln for ln in open(path) if ln.startswith("#")]
    for ln in open(path):
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        k, v = ln.split(":", 1)
        if k == "case":
            fx["case"].append(v.strip())
        else:
            fx[k] = v.strip()
    return fx, cite


def vec(s):
    return [float(t) for t in s.split()]


def rows(s):
    return [vec(r) for r in s.split(";")]


def quad(fx):
    return O.OracleProblem(O.MODEL_QUADRATIC, M=1, gamma=float(fx["gamma"]), noise_s=0.0,
                           h=vec(fx["h"]), xstar=vec(fx["xstar"]))


def test_every_fixture_is_cited():
    assert len(FILES) >= 8
    for p in FILES:
        fx, cite = parse(p)
        assert cite and any(("P:" in c or "S:" in c) for c in cite), p
        assert "kind" in fx, p


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(p) for p in FILES])
def test_golden(path):
    fx, _ = parse(path)
    kind, tol = fx["kind"], float(fx.get("tol", "0"))
    if kind == "replay":
        X0 = [[v] for v in vec(fx["X0"])]
        n = len(X0)
        if "ring" in fx:
            edges, role = synth.ring(int(fx["ring"]))
        else:
            edges, role = np.zeros((0, 2), np.int32), None
        if "repeat" in fx:
            events = [[int(t) for t in fx["repeat_event"].split()]] * int(fx["repeat"])
        else:
            events = [[int(t) for t in r.split()] for r in fx["events"].split(";")]
        X, _ = O.replay(quad(fx), X0, edges, role, events, T=int(fx.get("T", "0")))
        got = X[:n, 0]
        assert np.abs(got.astype(np.float64) - vec(fx["want"])).max() <= tol
        if "want_bits" in fx:
            bits = [int(b, 16) for b in fx["want_bits"].split()]
            assert [int(np.float32(v).view(np.uint32)) for v in got] == bits
    elif kind == "dpsgd":
        edges = [[int(t) for t in r.split()] for r in fx["edges"].split(";")]
        X = O.dpsgd_round(quad(fx), [[v] for v in vec(fx["X0"])], edges)
        assert np.abs(X[:, 0].astype(np.float64) - vec(fx["want"])).max() <= tol
    elif kind == "allreduce":
        x = O.allreduce_update(vec(fx["x"]), rows(fx["grads"]), float(fx["gamma"]))
        assert np.abs(np.asarray(x, np.float64) - vec(fx["want"])).max() <= tol
    elif kind == "pair_matrix":
        for c in fx["case"]:
            ijn, want = c.split("|")
            i, j, n = (int(t) for t in ijn.split())
            assert np.array_equal(TH.pair_matrix(i, j, n), np.array(rows(want)))
    elif kind == "expected_gram":
        for c in fx["case"]:
            n, e, want, rho = c.split("|")
            edges = [[int(t) for t in r.split()] for r in e.split(";")]
            g = TH.expected_gram(int(n), edges)
            assert np.abs(g - np.array(rows(want))).max() <= tol
            assert abs(TH.rho(g) - float(rho)) <= 1e-12
    else:
        pytest.fail(f"unknown fixture kind {kind}")
