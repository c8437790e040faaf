"""bench.py --gpus N launch logic (CPU): N ranks or a loud failure, never a
silent single-GPU run; both arms report the same config dict."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_single_gpu_runs_directly():
    assert bench.launch_plan(1, {}, 1) == ("direct", 1)


def test_multi_gpu_spawns_one_rank_per_gpu():
    assert bench.launch_plan(8, {}, 8) == ("spawn", 8)
    assert bench.launch_plan(2, {}, 8) == ("spawn", 2)


def test_too_few_gpus_fails_loudly():
    with pytest.raises(SystemExit):
        bench.launch_plan(2, {}, 1)
    with pytest.raises(SystemExit):
        bench.launch_plan(4, {"WORLD_SIZE": "4"}, 2)


def test_under_torchrun_world_must_match():
    assert bench.launch_plan(4, {"WORLD_SIZE": "4"}, 8) == ("rank", 4)
    with pytest.raises(SystemExit):
        bench.launch_plan(8, {"WORLD_SIZE": "4"}, 8)


def test_reference_arm_needs_no_gpu():
    assert bench.launch_plan(8, {}, 0, impl="reference") == ("direct", 1)
    assert bench.launch_plan(8, {"WORLD_SIZE": "8"}, 0, impl="reference") == ("rank", 8)


def test_seeds_and_config_shared_by_both_arms():
    assert bench.run_seeds(0)[0] == 1_000_000 and bench.run_seeds(1)[0] == 1_000_100
    assert bench.bench_config(2) == bench.bench_config(2)
    assert "seeds" in bench.bench_config(1)
