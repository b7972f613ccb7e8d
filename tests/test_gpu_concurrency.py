"""Concurrent solves of independent problems (SURVEY.md §8b threading: the
reference allows concurrent solves on different instances).  Each
Solver owns its context and stream; the cooperative loop launches of two
contexts on one device serialize on the hardware, so threads only interleave
-- the results must equal the sequential ones bit for bit."""
from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_2407_16144_b200 import hplp
from tests.helpers import csr_args
from tests.test_gpu_parity import std

pytestmark = pytest.mark.gpu


def test_threads_solve_independent_problems(gpu_required):
    names = ["cfg0", "cfg1_small", "zipf_small", "cfg0"]
    kw = dict(iteration_limit=3000, tolerance=1e-12)
    seq = [hplp.solve(*csr_args(std(nm)[1]), **kw) for nm in names]
    out = [None] * len(names)
    err = []

    def work(k):
        try:
            sol = hplp.Solver(*csr_args(std(names[k])[1]))
            try:
                for _ in range(2):  # repeated solves on one context, interleaved with the others
                    out[k] = sol.solve(**kw)
            finally:
                sol.close()
        except Exception as e:  # noqa: BLE001 -- reported below
            err.append(e)

    for nm in names:  # problems built before the threads start (the cache is not thread-safe)
        std(nm)
    ts = [threading.Thread(target=work, args=(k,)) for k in range(len(names))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not err, err
    for a, b in zip(out, seq):
        assert a["iterations"] == b["iterations"] and a["status"] == b["status"]
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
        assert [e[:2] for e in a["epochs"]] == [e[:2] for e in b["epochs"]]
