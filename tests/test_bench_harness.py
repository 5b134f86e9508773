"""bench.py harness logic on the CPU: block-aligned shard ranges and the
strong-scaling snapshot generator (configs[4]) — the shards of any rank
count concatenate to the same global dataset."""

import sys

import torch

import bench


def test_shard_ranges_are_block_aligned_and_cover():
    for total in (1, 1023, 1024, 5000, 2_000_000_000):
        for world in (1, 2, 3, 4, 8):
            r = [bench.shard_range(total, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == total
            for (a, b), (c, _) in zip(r, r[1:]):
                assert b == c and (b - a) % 1024 == 0


def test_snapshot_shards_concatenate_to_the_same_dataset(monkeypatch):
    monkeypatch.setattr(bench, "SHARD_CHUNK", 1 << 14)
    total = 3 * (1 << 14) + 777
    cpu = torch.device("cpu")
    pos1, vel1 = bench.gen_snapshot_shard(total, 0, total, 7, cpu)
    for world in (2, 3, 4):
        parts = [bench.gen_snapshot_shard(total, *bench.shard_range(total, world, k), 7, cpu) for k in range(world)]
        for a in range(3):
            assert torch.equal(torch.cat([p[0][a] for p in parts]), pos1[a])
            assert torch.equal(torch.cat([p[1][a] for p in parts]), vel1[a])


def test_workloads_name_the_baseline_configs():
    assert sorted(w["config"] for w in bench.WORKLOADS.values()) == [1, 2, 3, 4]
    assert bench.WORKLOADS["snapshot2b"]["scaling"] == "strong"
    assert sys.modules["bench"].PARTICLES == 280_000_000
