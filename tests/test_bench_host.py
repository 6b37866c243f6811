"""Host logic of the bench and the sweep harness (-m "not gpu"): the launch a run uses is
the one the parity tests pin (bench.launch_of / TPCC_CONFIGS), and the launch count the
JSON line claims follows the library's per-submit kernel sequence."""
import types

import bench


def test_ycsb_launch_is_one_txn_per_warp_tuned():
    a = types.SimpleNamespace(launch="tuned", lanes=32, wd=0, bs=32)
    for s, bs in bench.TUNED_BS.items():
        assert bench.launch_of(a, s, 148) == {"wd": 0, "bs": bs, "grid": 148}
        assert 1 <= bs <= 32   # one block of bs warps per SM (<= 1,024 threads)
    a16 = types.SimpleNamespace(launch="tuned", lanes=16, wd=0, bs=32)
    assert bench.launch_of(a16, "gacco", 148)["bs"] == bench.TUNED_BS_16["gacco"]
    # the paper's launch: thread mode, full-occupancy grid, the given (wd, bs)
    t = types.SimpleNamespace(launch="tuned", lanes=1, wd=5, bs=8)
    assert bench.launch_of(t, "tpl_nw", 148) == {"wd": 5, "bs": 8, "grid": 0}
    f = types.SimpleNamespace(launch="fixed", lanes=32, wd=0, bs=16)
    assert bench.launch_of(f, "to", 148) == {"wd": 0, "bs": 16, "grid": 0}


def test_tpcc_configs_cover_every_scheme():
    names = [c["name"] for c in bench.TPCC_CONFIGS]
    assert [c["W"] for c in bench.TPCC_CONFIGS] == [1, 64, 512] and len(set(names)) == 3
    for c in bench.TPCC_CONFIGS:
        for s in ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]:
            bs, one_block = c["launch"].get(s, c["launch"]["*"])
            assert bs >= 1 and isinstance(one_block, bool)


def test_launch_count_follows_the_submit_sequence():
    # a1 generator + per scheme: a2 (1) + exec (1) + copy-out with stats (1) + commit
    # positions + the background zeroing kernel of the non-deterministic schemes
    s2 = bench.launches_per_step(["tpl_nw"])
    assert s2 == 1 + 1 + 1 + 1 + 0 + 1
    assert bench.launches_per_step(["to"]) == 1 + 1 + 1 + 1 + 5 + 1
    assert bench.launches_per_step(["tictoc"]) == 1 + 1 + 1 + 1 + 4 + 1
    assert bench.launches_per_step(["tpl_nw", "to"]) == s2 + (1 + 1 + 1 + 5 + 1)
    # a prepared (pipelined) deterministic submit adds one error merge; its a3 still runs
    # inside the step (on the prep stream)
    assert bench.launches_per_step(["gacco"], pipelined=True) == bench.launches_per_step(["gacco"]) + 1
    assert bench.launches_per_step(["gputx"]) > bench.launches_per_step(["gacco"])


def test_sweep_bench_mode_matches_the_bench_launch():
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import sweep
    db = types.SimpleNamespace(num_sms=148)
    assert sweep.mode_kw("bench", "mvcc", db) == dict(lanes=32, wd=0, bs=bench.TUNED_BS["mvcc"], grid=148)
    assert sweep.mode_kw(dict(lanes=1, wd=0, bs=32), "mvcc", db) == dict(lanes=1, wd=0, bs=32)
