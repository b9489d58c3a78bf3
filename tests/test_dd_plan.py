"""Host logic of the spatial DD (no GPU): partition plans against the
reference's plans (dist.py:104-127, golden ranges from the reference run),
the reduced-chain node list (dist.py:476-483) and the throughput plan."""

import pytest

from paper_2508_19138_b200.dd import PartitionError, PartitionPlan, balanced_partition_plan, make_partition_plan


def test_plans_match_reference(golden):
    g = golden("golden_dd.npz")
    for c in range(int(g["n_cases"])):
        seed, nb, bs, p_s = (int(x) for x in g[f"c{c}_cfg"])
        assert [list(r) for r in make_partition_plan(nb, p_s).ranges] == g[f"c{c}_ranges"].tolist()


def test_plan_validation_and_nodes():
    p = make_partition_plan(12, 4)
    assert p.nodes() == [2, 3, 5, 6, 8, 9]
    assert p.p_s == 4 and p.width(1) == 3
    with pytest.raises(PartitionError):
        make_partition_plan(5, 3)
    with pytest.raises(PartitionError):
        PartitionPlan(6, ((0, 2), (4, 5)))
    with pytest.raises(PartitionError):
        PartitionPlan(6, ((0, 0), (1, 5)))


@pytest.mark.parametrize("n,p", [(32, 3), (32, 4), (32, 8), (40, 8), (17, 4), (9, 4)])
def test_balanced_plan_tiles_the_chain(n, p):
    plan = balanced_partition_plan(n, p)
    assert plan.n_blocks == n and plan.p_s == p
    widths = [b - a + 1 for a, b in plan.ranges]
    assert min(widths) >= 2 and sum(widths) == n
    if p > 2 and widths != [b - a + 1 for a, b in make_partition_plan(n, p).ranges]:
        assert widths[0] >= max(widths[1:-1])
