"""CPU: the 1F1B schedule of pipeline.py — every stage runs each micro-batch's forward before its
backward, the stages' orders are mutually consistent (a discrete-event run with blocking receives
and buffered sends completes: no deadlock), at most min(P - s, m) micro-batches are in flight on
stage s (the activation slots), and the traced boundary volume 2 (P - 1) b s d relates to the
reference's closed form 2 p b s d (costs.py:63-64)."""

import pytest

from paper_2512_12131_b200.model import ModelConfig, RunShape
from paper_2512_12131_b200.pipeline import pp_boundary_elements, schedule_1f1b


def _simulate(P, m):
    """Event-driven execution: F(j) on stage s > 0 needs the activation from stage s-1, B(j) on
    stage s < P-1 needs the gradient from stage s+1; sends never block."""
    sched = {s: schedule_1f1b(s, P, m) for s in range(P)}
    pos = {s: 0 for s in range(P)}
    act, grad = set(), set()  # (stage_from, j) messages delivered
    done = 0
    total = sum(len(v) for v in sched.values())
    in_flight = {s: 0 for s in range(P)}
    peak = {s: 0 for s in range(P)}
    while done < total:
        progressed = False
        for s in range(P):
            if pos[s] == len(sched[s]):
                continue
            op, j = sched[s][pos[s]]
            if op == "F":
                if s > 0 and (s - 1, j) not in act:
                    continue
                act.add((s, j))
                in_flight[s] += 1
                peak[s] = max(peak[s], in_flight[s])
            else:
                if s < P - 1 and (s + 1, j) not in grad:
                    continue
                grad.add((s, j))
                in_flight[s] -= 1
            pos[s] += 1
            done += 1
            progressed = True
        if not progressed:
            raise AssertionError(f"deadlock at {pos}")
    return peak


@pytest.mark.parametrize("P,m", [(1, 1), (1, 4), (2, 1), (2, 4), (4, 4), (4, 8), (8, 3), (8, 16)])
def test_1f1b_is_complete_consistent_and_bounded(P, m):
    for s in range(P):
        sch = schedule_1f1b(s, P, m)
        assert sorted(j for op, j in sch if op == "F") == list(range(m))
        assert sorted(j for op, j in sch if op == "B") == list(range(m))
        for j in range(m):
            assert sch.index(("F", j)) < sch.index(("B", j))
    peak = _simulate(P, m)
    for s in range(P):
        assert peak[s] <= min(P - s, m)


def test_1f1b_warmup_counts():
    assert schedule_1f1b(0, 4, 8)[:4] == [("F", 0), ("F", 1), ("F", 2), ("F", 3)]
    assert schedule_1f1b(3, 4, 8)[:2] == [("F", 0), ("B", 0)]
    with pytest.raises(ValueError):
        schedule_1f1b(2, 2, 4)


def test_boundary_volume_vs_reference_closed_form():
    cfg = ModelConfig(layers=4, heads=4, d=256, d_ff=640, r=64)
    shape = RunShape(4, 64, 2, 2)
    # 2 (P - 1) b s d traced; the reference's iter_volume("pp") = 2 p b s d (costs.py:63-64)
    assert pp_boundary_elements(cfg, shape, 2) == 2 * 1 * 4 * 64 * 256
    assert pp_boundary_elements(cfg, shape, 2) * shape.p == (shape.p - 1) * 2 * shape.p * 4 * 64 * 256
