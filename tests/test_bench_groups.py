"""bench.py's rank grouping for --gpus N --tp P (configs[3]): TP groups are P consecutive ranks, DP groups join the
ranks with the same TP rank, every rank is in exactly one group of each kind, and each group's NCCL-id root is a
member of it (CPU only: no NCCL is created)."""
import pytest

import bench


@pytest.mark.parametrize("world,tp", [(1, 1), (2, 1), (2, 2), (4, 2), (8, 2), (8, 4), (8, 8)])
def test_rank_groups_partition(world, tp):
    g = [bench.rank_groups(r, world, tp) for r in range(world)]
    tp_groups, dp_groups = {}, {}
    for r, (tr, dr, dw, troot, droot) in enumerate(g):
        assert dw == world // tp and r == dr * tp + tr
        tp_groups.setdefault(troot, []).append((tr, r))
        dp_groups.setdefault(droot, []).append((dr, r))
    assert len(tp_groups) == world // tp and len(dp_groups) == tp
    for root, mem in tp_groups.items():
        assert sorted(t for t, _ in mem) == list(range(tp)) and root in [r for _, r in mem]
        assert [r for _, r in sorted(mem)] == list(range(root, root + tp))  # consecutive ranks
    for root, mem in dp_groups.items():
        assert sorted(d for d, _ in mem) == list(range(world // tp)) and root in [r for _, r in mem]


def test_rank_groups_rejects_bad_tp():
    with pytest.raises(ValueError):
        bench.rank_groups(0, 6, 4)
