"""Reentrancy (evaluate is pure and reentrant; concurrent calls on
disjoint inputs are allowed): one context per thread, calls racing on the device,
results bitwise equal to the same calls made serially; errors stay per thread
(hmdp_last_error is thread-local)."""
import threading

import numpy as np
import pytest

import paper_2602_02234_b200 as P

pytestmark = pytest.mark.gpu


def _jobs(golden_models):
    jobs = []
    for k, (name, n) in enumerate([("dpa3", 582), ("dpa2", 1231), ("dpa3", 1231), ("dpa2", 582)]):
        s = P.generate_synthetic_system(n, seed=7 + k)
        jobs.append((P.model_from_json(golden_models[name]), s))
    return jobs


def test_concurrent_contexts_match_serial(golden_models):
    jobs = _jobs(golden_models)
    serial = []
    for m, s in jobs:
        ctx = P.Context(m)
        serial.append([ctx.compute(s.positions, s.types, s.box, prec) for prec in
                       (P.Precision.fp32, P.Precision.fp64)])
        ctx.close()
    out = [None] * len(jobs)
    errs = []

    def work(k):
        try:
            m, s = jobs[k]
            ctx = P.Context(m)
            res = []
            for _ in range(20):  # repeated: the cached-graph path races too
                res = [ctx.compute(s.positions, s.types, s.box, prec) for prec in
                       (P.Precision.fp32, P.Precision.fp64)]
            out[k] = res
            ctx.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a, b in zip(out, serial):
        for x, y in zip(a, b):
            assert x.energy == y.energy
            assert np.array_equal(x.forces, y.forces)
            assert np.array_equal(x.virial_tensor, y.virial_tensor)


def test_errors_stay_on_their_thread(golden_models):
    """A failing call on one thread does not leak its message into another's."""
    m = P.model_from_json(golden_models["dpa2"])
    s = P.generate_synthetic_system(582)
    msgs = {}

    def bad():
        ctx = P.Context(m)
        try:
            ctx.compute(s.positions, np.full(582, 7, dtype=np.int32), s.box)
        except ValueError as e:
            msgs["bad"] = str(e)

    def good():
        ctx = P.Context(m)
        for _ in range(10):
            ctx.compute(s.positions, s.types, s.box)
        msgs["good"] = "ok"

    th = [threading.Thread(target=bad), threading.Thread(target=good)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert msgs.get("good") == "ok"
    assert "out of range" in msgs.get("bad", "")
