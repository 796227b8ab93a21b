"""The paper's progressive-allocation deadlock (PAPER.md P:340-351,
fig:deadlock) reproduced in the oracle, and Salus's lanes avoiding it."""
from oracle import deadlock as D


def test_paper_example_deadlocks_without_lanes():
    # C = 12 GB, P_A = P_B = 1 GB, E_A = E_B = 7 GB allocated in increments;
    # after (P_A, P_B, E_A += 4, E_B += 4) both need 3 GB more with 2 GB free
    steps = [("A", "P", 1), ("B", "P", 1), ("A", "E", 4), ("B", "E", 4), ("A", "E", 3), ("B", "E", 3)]
    res, pend = D.progressive(12, steps)
    assert res == "deadlock"
    assert pend == {"A": ("E", 3), "B": ("E", 3)}      # "(E_A += 3 GB) and (E_B += 3 GB)"


def test_same_demand_allocated_up_front_completes():
    # the same two iterations, each allocating its whole E at once: no deadlock
    steps = [("A", "P", 1), ("B", "P", 1), ("A", "E", 7), ("B", "E", 7)]
    assert D.progressive(12, steps)[0] == "done"


def test_lanes_admit_both_into_one_serialised_lane():
    # Salus: 1 + 1 + 7 <= 12 -> A opens a lane of 7, B joins it (branch 2);
    # their iterations run one at a time inside 7 GB: never a deadlock
    res, admitted, lanes, waiting = D.with_lanes(12, [("A", 1, 7), ("B", 1, 7)])
    assert res == "done" and admitted == ["A", "B"] and lanes == [["A", "B"]] and waiting == []
