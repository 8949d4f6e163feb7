"""bench.py's host-side accounting (no GPU): the padding-waste and sine-roofline figures it prints are
checked against hand counts, so a wrong tile size, padded width or layer count in them fails here."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_padding_waste_hand_counts():
    # 512 depth-2 points and 256 depth-3 points fill whole 256-row tiles: nothing padded at H = 256
    w = bench._padding_waste([7, 0, 512, 256], 256, False)
    assert w["tile_rows"] == 256 and w["padded_width"] == 256
    assert w["waste_frac"] == 0.0
    # depth-1 points carry no H x H layer, so they never count; 1 depth-2 point pads a 256-row tile
    w = bench._padding_waste([0, 1000, 1], 256, False)
    assert w["executed_flops"] == 256 * 2.0 * 256 * 256
    assert w["waste_frac"] == pytest.approx(255 / 256)
    # H = 336 runs at the padded width 352 (zero weights): waste 1 - (336/352)^2 on full tiles
    w = bench._padding_waste([0, 0, 256], 336, False)
    assert w["padded_width"] == 352
    assert w["waste_frac"] == pytest.approx(1 - (336 / 352) ** 2)
    # the FP32 path: 128-row tiles, no width padding
    w = bench._padding_waste([0, 0, 129], 336, True)
    assert (w["tile_rows"], w["padded_width"]) == (128, 336)
    assert w["waste_frac"] == pytest.approx(1 - 129 / 256)
    # slot-team kernel: every depth bucket padded to an even number of 256-row tiles (3 tiles -> 4, 2 stay 2)
    w = bench._padding_waste([0, 0, 3 * 256, 2 * 256], 256, False, even_bins=True)
    assert w["executed_flops"] == 4 * 256 * 2.0 * 256 * 256 + 2 * 256 * 2 * 2.0 * 256 * 256
    assert w["waste_frac"] == pytest.approx(1 - (3 * 1 + 2 * 2) / (4 * 1 + 2 * 2))


def test_sine_roofline_counts_every_evaluated_layer():
    # Eq. 2: a depth-d point evaluates sin on H units in each of its d layers (layer 1 included);
    # depth-0 points (cached far-field SDF) evaluate none
    r = bench._sine_roofline([5, 10, 20, 0, 1], 64, 2.0, {"sm_mhz": 1000.0})
    assert r["sines_per_launch"] == (10 * 1 + 20 * 2 + 1 * 4) * 64
    assert r["achieved"] == pytest.approx(r["sines_per_launch"] / 2e-3 / 1e9)
    assert r["peak"] == pytest.approx(148 * 16 * 1e9 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])


def test_reference_arm_config_equals_this_arms():
    """The driver compares the two arms' lines: at N = 1 the reference arm's `config` must be the one
    this arm prints (same workload string as the z-slab shard of rank 0 of 1)."""
    import argparse
    from paper_2604_25936_b200 import partition
    import sandgen as g
    args = argparse.Namespace(config="C2", full_depth=False, scaling="strong")
    c = g.make_config("C2")
    k0, k1, Rz = partition.shard_planes(c.depthmap, c.grid_R, 1, 0, weak=False)
    wl_this = f"C2: {c.grid_R}x{c.grid_R}x{Rz} grid, z-planes [{k0},{k1}) on rank 0"
    assert bench._n1_workload(args, c) == wl_this
    this = bench._arm_config(args, c, 1, wl_this, c.grid_R ** 3)
    ref = bench._arm_config(args, c, 1, bench._n1_workload(args, c), c.grid_R ** 3)
    assert this == ref
    assert this["global_points"] == 512 ** 3 and "no flush needed" in this["l2"]


def test_c4_strong_config_line():
    """N > 1 default: C4's fixed 1024^3 grid (global_points 1024^3 for any N), strong-scaled."""
    import argparse
    import sandgen as g
    args = argparse.Namespace(config="C4", full_depth=False, scaling="strong")
    c = g.make_config("C4")
    cfg = bench._arm_config(args, c, 8, "unused", c.grid_R ** 3)
    assert cfg["global_points"] == 1024 ** 3 and "strong-scaled" in cfg["workload"]
    assert cfg["parallelism"] == "dp8 (z-slab shards)" and "level-8" in cfg["depth_map"]


def test_gpus_flag_relaunches_and_rejects_mismatch(monkeypatch):
    """--gpus N without a torchrun environment re-executes under torch.distributed.run with N ranks; a
    torchrun environment whose WORLD_SIZE differs from --gpus is an error (never a silent 1-rank run)."""
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.os, "execv", lambda exe, cmd: calls.append(cmd) or (_ for _ in ()).throw(SystemExit(0)))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit):
        bench.main()
    cmd = calls[0]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4"])
    with pytest.raises(SystemExit) as e:
        bench.main()
    assert "WORLD_SIZE" in str(e.value)
