"""-m gpu: parity of the CUDA path (through the C ABI) against the CPU oracle on YCSB.

Bar: bit-exact.  For every scheme the GPU's read outputs and final
table equal the oracle's serial replay of the committed set in the GPU-reported order;
GPUTx and GaccO must also report ascending batch order with zero aborts."""
import numpy as np
import pytest

import inputs

pytestmark = pytest.mark.gpu

SCHEMES = ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc", "gputx", "gacco"]


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.fixture(scope="module")
def c1(torch_cuda, orc):
    """BASELINE.json configs[0]: 1,024 rows, 1,024 txns x 4 ops, W=0.5, theta=0.8."""
    from paper_2406_10158_b200.api import DB
    db = DB(0)
    db.load_ycsb(1024, 11)
    S0 = db.read_table(0)
    db.snapshot(True)
    yield db, S0
    db.close()


def test_device_rows_equal_input_generator(c1):
    db, S0 = c1
    assert np.array_equal(S0, inputs.ycsb_rows(11, 1024))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_a1_generator_bitexact(c1, orc, seed):
    db, _ = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, seed, T, A)
    k, o = b.export_ycsb()
    ek, eo = orc.ycsb_gen(seed, 1024, 1024, 4, 0.5, T, A)
    assert np.array_equal(k, ek) and np.array_equal(o, eo)
    b.free()


# (wd, bs, lanes): thread mode corners of the paper's launch grid + tile modes
CORNERS = [(0, 32, 1), (5, 1, 1), (0, 1, 1), (5, 32, 1), (2, 8, 1), (0, 32, 4), (0, 8, 8), (0, 32, 16), (0, 8, 32)]


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("wd,bs,lanes", CORNERS)
def test_c1_parity(c1, orc, scheme, wd, bs, lanes):
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    for seed in (5, 6):
        b = db.gen_ycsb(1024, 4, 0.5, seed, T, A)
        keys, ops = orc.ycsb_gen(seed, 1024, 1024, 4, 0.5, T, A)
        db.snapshot(False)
        res = db.submit(b, scheme, wd=wd, bs=bs, lanes=lanes)
        st = db.sync()
        assert st.commits == 1024
        h = res.host(db.stream)
        assert int(h["restarts"].astype(np.int64).sum()) == st.aborts
        orc.check_ycsb(scheme, S0, keys, ops, 4, h, db.read_table(0))
        if scheme == "gputx":
            assert st.max_rank == int(orc.gputx_ranks(keys, ops, 4, 1024).max())
        b.free()


@pytest.mark.parametrize("lanes", [1, 4])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_immediate_retry_mode(c1, orc, scheme, lanes):
    from paper_2406_10158_b200.gcctb import CC_FLAG_IMMEDIATE_RETRY
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 9, T, A)
    keys, ops = orc.ycsb_gen(9, 1024, 1024, 4, 0.5, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=32, flags=CC_FLAG_IMMEDIATE_RETRY, lanes=lanes)
    db.sync()
    orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("lanes", [1, 4])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_read_only_never_aborts(c1, orc, scheme, lanes):
    """RO preset: no scheme aborts, state unchanged."""
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.99)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.0, 3, T, A)
    keys, ops = orc.ycsb_gen(3, 1024, 1024, 4, 0.0, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=5, bs=32, lanes=lanes)
    st = db.sync()
    assert st.aborts == 0
    h = res.host(db.stream)
    orc.check_ycsb(scheme, S0, keys, ops, 4, h, db.read_table(0))
    assert np.array_equal(db.read_table(0), S0)
    b.free()


@pytest.mark.parametrize("scheme", SCHEMES)
def test_brute_force_tiny(c1, orc, scheme):
    """<=7 txns x <=3 ops over <=5 rows, W=0.5: the GPU outcome is one of the n! serial
    outcomes, and the reported order reproduces it."""
    db, S0 = c1
    rng = np.random.default_rng(1234 + len(scheme))
    for it in range(40):
        n = int(rng.integers(2, 8))
        k = int(rng.integers(1, 4))
        keys, ops = inputs.random_batch(int(rng.integers(1 << 30)), n, k, 1024, 0.5, hot=5)
        b = db.import_ycsb(keys, ops, k)
        db.snapshot(False)
        lanes = [1, 4][it % 2]
        res = db.submit(b, scheme, wd=int(rng.integers(0, 6)), bs=int(rng.integers(1, 5)), lanes=lanes)
        db.sync()
        h = res.host(db.stream)
        after = db.read_table(0)
        orc.check_ycsb(scheme, S0, keys, ops, k, h, after)
        outs = orc.ycsb_serial_outcomes(S0[:5].copy(), keys, ops, k, list(range(n)))
        got = (after[:5].tobytes(), h["read_out"].reshape(n, k).tobytes())
        assert got in outs
        b.free()


@pytest.mark.parametrize("scheme,lanes", [("silo", 1), ("silo", 4), ("gacco", 1), ("gacco", 4), ("gputx", 4)])
def test_key_not_found(c1, scheme, lanes):
    """KeyNotFound is reported, also when a3 resolves the keys (GaccO / GPUTx:
    no out-of-range record reaches the executor), and the db stays usable."""
    from paper_2406_10158_b200.gcctb import CCError
    db, _ = c1
    b = db.import_ycsb(np.array([1, 5000, 7, 9], np.uint32), np.array([0, 0, 0x80, 0], np.uint8), 2)
    db.submit(b, scheme, lanes=lanes)
    with pytest.raises(CCError, match="KEY_NOT_FOUND"):
        db.sync()
    b.free()
    b = db.import_ycsb(np.array([1, 2, 7, 9], np.uint32), np.array([0, 0, 0x80, 0], np.uint8), 2)
    db.snapshot(False)
    db.submit(b, scheme, lanes=lanes)
    assert db.sync().commits == 2
    b.free()


@pytest.fixture(scope="module")
def c2(torch_cuda, orc):
    """BASELINE.json configs[1]: 10,485,760-row table, 64K x 16 ops."""
    from paper_2406_10158_b200.api import DB
    n = 10 * (1 << 20)
    db = DB(0)
    db.load_ycsb(n, 5)
    S0 = db.read_table(0)
    assert np.array_equal(S0[:4096], inputs.ycsb_rows(5, 4096))
    assert np.array_equal(S0[-4096:], inputs.ycsb_rows(5, 4096, n - 4096))
    db.snapshot(True)
    yield db, S0, n
    db.close()


# full size: the paper's launch (thread mode, wd=0, bs=32) across the theta range, and
# tile mode (16 lanes) in the full-occupancy grid; the bench's own per-scheme launch is
# covered up to theta=0.99 by test_c2_full_size_parity_bench_launch.
C2_CASES = [(0.0, 1), (0.6, 1), (0.99, 1), (0.6, 16), (0.9, 16), (0.99, 16)]


@pytest.mark.parametrize("theta,lanes", C2_CASES)
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c2_full_size_parity(c2, orc, scheme, theta, lanes):
    """Full-size parity (BASELINE.json configs[1]) in the bench launch configurations."""
    db, S0, n = c2
    T = inputs.zipf_thresholds(n, theta)
    A = inputs.scramble_mult(n)
    B, K, W = 1 << 16, 16, 0.1
    b = db.gen_ycsb(B, K, W, 77, T, A)
    keys, ops = orc.ycsb_gen(77, n, B, K, W, T, A)
    k2, o2 = b.export_ycsb()
    assert np.array_equal(keys, k2) and np.array_equal(ops, o2)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes, watchdog_s=60)
    st = db.sync()
    assert st.commits == B
    orc.check_ycsb(scheme, S0, keys, ops, K, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("theta,warm", [(0.6, False), (0.6, True), (0.9, False), (0.9, True),
                                        (0.95, False), (0.99, False)])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c2_full_size_parity_bench_launch(c2, orc, scheme, theta, warm):
    """configs[1] at full size in exactly the launch bench.py times (bench.launch_of: one
    transaction per warp -- 32-lane tiles, 16 lanes idle at K = 16 -- per-scheme warps per
    SM, one block per SM), at the bench's theta and above."""
    import types
    import bench
    db, S0, n = c2
    a = types.SimpleNamespace(launch="tuned", lanes=32, wd=0, bs=32)
    la = bench.launch_of(a, scheme, db.num_sms)
    assert la["grid"] == db.num_sms
    T = inputs.zipf_thresholds(n, theta)
    A = inputs.scramble_mult(n)
    B, K, W = 1 << 16, 16, 0.1
    b = db.gen_ycsb(B, K, W, 79, T, A)
    keys, ops = orc.ycsb_gen(79, n, B, K, W, T, A)
    db.snapshot(False)
    from paper_2406_10158_b200.gcctb import CC_FLAG_WARM
    res = db.submit(b, scheme, lanes=32, watchdog_s=60, flags=CC_FLAG_WARM if warm else 0, **la)
    st = db.sync()
    assert st.commits == B
    orc.check_ycsb(scheme, S0, keys, ops, K, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("mode", ["meta_pad", "meta_pad_latched"])
@pytest.mark.parametrize("lanes", [1, 16])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c1_parity_layout_flags(c1, orc, scheme, lanes, mode):
    """CC_FLAG_META_PAD (one control word per 32 B sector, f-3) -- also under latched
    words, whose latch index follows the word -- changes the memory layout only: the
    same serial-replay parity at configs[0]."""
    from paper_2406_10158_b200 import gcctb as G
    flags = {"meta_pad": G.CC_FLAG_META_PAD, "meta_pad_latched": G.CC_FLAG_META_PAD | G.CC_FLAG_LATCHED}[mode]
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 23, T, A)
    keys, ops = orc.ycsb_gen(23, 1024, 1024, 4, 0.5, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=5 if lanes == 1 else 0, bs=8, lanes=lanes, flags=flags)
    assert db.sync().commits == 1024
    orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("lanes", [4, 8, 16])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c1_parity_warm(c1, orc, scheme, lanes):
    """CC_FLAG_WARM (wait for the lines to reach L2 before the first CC step) changes
    timing only: same serial-replay parity at configs[0]."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_WARM
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 17, T, A)
    keys, ops = orc.ycsb_gen(17, 1024, 1024, 4, 0.5, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=8, lanes=lanes, flags=CC_FLAG_WARM)
    st = db.sync()
    assert st.commits == 1024
    orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("scheme", SCHEMES)
def test_c1_parity_warp_per_txn(c1, orc, scheme):
    """32-lane tiles (one warp per transaction, lanes >= K idle) give the oracle's results."""
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 46, T, A)
    keys, ops = orc.ycsb_gen(46, 1024, 1024, 4, 0.5, T, A)
    for bs, grid in ((32, 0), (4, 148)):
        db.snapshot(False)
        res = db.submit(b, scheme, bs=bs, grid=grid, lanes=32)
        db.sync()
        orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("lanes", [1, 4])
def test_c1_parity_mvcc_split_layout(c1, orc, lanes):
    """f-3 metadata ablation: MVCC with split timestamp / version-pointer arrays gives the
    same results as Table II's interleaved layout."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_MVCC_SPLIT
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 45, T, A)
    keys, ops = orc.ycsb_gen(45, 1024, 1024, 4, 0.5, T, A)
    db.snapshot(False)
    res = db.submit(b, "mvcc", wd=0, bs=32, lanes=lanes, flags=CC_FLAG_MVCC_SPLIT)
    db.sync()
    orc.check_ycsb("mvcc", S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


def test_c2_mvcc_split_layout(c2, orc):
    from paper_2406_10158_b200.gcctb import CC_FLAG_MVCC_SPLIT
    db, S0, n = c2
    T = inputs.zipf_thresholds(n, 0.9)
    A = inputs.scramble_mult(n)
    b = db.gen_ycsb(1 << 16, 16, 0.1, 79, T, A)
    keys, ops = orc.ycsb_gen(79, n, 1 << 16, 16, 0.1, T, A)
    db.snapshot(False)
    res = db.submit(b, "mvcc", wd=0, bs=32, lanes=16, flags=CC_FLAG_MVCC_SPLIT, watchdog_s=60)
    assert db.sync().commits == 1 << 16
    orc.check_ycsb("mvcc", S0, keys, ops, 16, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("flag", ["tree", "binary", "eytz"])
@pytest.mark.parametrize("scheme", ["tpl_nw", "tictoc", "gacco"])
def test_c2_full_size_parity_search_index(c2, orc, scheme, flag):
    """configs[1] in the bench launch with the search indexes (bench --index tree|binary|eytz)."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_INDEX_BINARY, CC_FLAG_INDEX_EYTZ, CC_FLAG_INDEX_TREE
    db, S0, n = c2
    T = inputs.zipf_thresholds(n, 0.6)
    A = inputs.scramble_mult(n)
    B, K, W = 1 << 16, 16, 0.1
    b = db.gen_ycsb(B, K, W, 78, T, A)
    keys, ops = orc.ycsb_gen(78, n, B, K, W, T, A)
    db.snapshot(False)
    fl = {"binary": CC_FLAG_INDEX_BINARY, "tree": CC_FLAG_INDEX_TREE, "eytz": CC_FLAG_INDEX_EYTZ}[flag]
    res = db.submit(b, scheme, wd=0, bs=32, lanes=16, flags=fl, watchdog_s=60)
    st = db.sync()
    assert st.commits == B
    orc.check_ycsb(scheme, S0, keys, ops, K, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("lanes", [1, 16])
@pytest.mark.parametrize("scheme", ["to", "mvcc"])
def test_ts_overflow_is_reported(c1, monkeypatch, scheme, lanes):
    """31-bit TO / MVCC timestamps: exhausting them
    surfaces as TS_OVERFLOW, never as a wrong result or a hang.  The counter starts 2,000
    below 2^31 (test hook GCCTB_TS_BASE) and 1,024 all-write transactions on 4 hot rows
    need far more than 2,000 attempts, so the overflow must be reported -- a watchdog
    expiry fails the test."""
    from paper_2406_10158_b200.gcctb import CCError
    db, S0 = c1
    keys = np.tile(np.arange(4, dtype=np.uint32), 1024)
    ops = np.full(keys.size, 0x81, np.uint8)
    b = db.import_ycsb(keys, ops, 4)
    db.snapshot(False)
    monkeypatch.setenv("GCCTB_TS_BASE", str((1 << 31) - 2000))
    db.submit(b, scheme, wd=5, bs=32, lanes=lanes, watchdog_s=20)
    with pytest.raises(CCError) as ei:
        db.sync()
    assert "TS_OVERFLOW" in str(ei.value)
    # the same batch from timestamp 1 commits every transaction correctly
    monkeypatch.delenv("GCCTB_TS_BASE")
    db.snapshot(False)
    res = db.submit(b, scheme, wd=5, bs=32, lanes=lanes, watchdog_s=60)
    assert db.sync().commits == 1024
    import oracle
    oracle.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("n", [1, 15, 16, 17, 255, 4097, 300001])
def test_index_lookup_tree_and_binary(torch_cuda, n):
    """the row of a present key, KeyNotFound (2^64-1) otherwise; the
    cache-line tree and the paper's binary search agree with numpy.searchsorted."""
    from paper_2406_10158_b200.api import DB
    rng = np.random.default_rng(n)
    keys = np.unique(rng.integers(0, 1 << 62, size=n * 2, dtype=np.uint64))[:n]
    keys.sort()
    n = keys.size
    rows = rng.permutation(n).astype(np.uint64)
    db = DB(0)
    tid = db.create_table("t", 8, n)
    iid = db.create_index(tid, keys, rows)
    probe = np.concatenate([keys, keys + np.uint64(1), np.array([0, (1 << 63)], np.uint64), keys[:3] - np.uint64(1)])
    pos = np.searchsorted(keys, probe)
    hit = (pos < n) & (keys[np.minimum(pos, n - 1)] == probe)
    exp = np.where(hit, rows[np.minimum(pos, n - 1)], np.uint64((1 << 64) - 1))
    for method in ("auto", "tree", "binary", "eytz"):
        got = db.index_lookup(iid, probe, method=method)
        assert np.array_equal(got, exp), method
    db.close()


@pytest.mark.parametrize("k0,n,identity", [(0, 1, True), (0, 17, True), (5, 4097, False), ((1 << 40) + 3, 300001, False),
                                           (0, 300001, True), (0, 300001, False)])
def test_index_lookup_dense(torch_cuda, k0, n, identity):
    """f-3 direct addressing: on a dense key range k0..k0+n-1 the default lookup (no probe)
    returns what numpy.searchsorted does, just outside the range too."""
    from paper_2406_10158_b200.api import DB
    rng = np.random.default_rng(n + k0)
    keys = np.uint64(k0) + np.arange(n, dtype=np.uint64)
    rows = np.arange(n, dtype=np.uint64) if identity else rng.permutation(n).astype(np.uint64)
    db = DB(0)
    tid = db.create_table("t", 8, n)
    iid = db.create_index(tid, keys, rows)
    probe = np.concatenate([keys, rng.choice(keys, 1000), keys[-1:] + np.uint64(1), keys[-1:] + np.uint64(1 << 33),
                            np.array([0, 1, (1 << 63), (1 << 64) - 2], np.uint64)])
    if k0:
        probe = np.concatenate([probe, np.array([k0 - 1], np.uint64)])
    pos = np.searchsorted(keys, probe)
    hit = (pos < n) & (keys[np.minimum(pos, n - 1)] == probe)
    exp = np.where(hit, rows[np.minimum(pos, n - 1)], np.uint64((1 << 64) - 1))
    for method in ("auto", "tree", "binary", "eytz"):
        assert np.array_equal(db.index_lookup(iid, probe, method=method), exp), method
    db.close()


@pytest.mark.parametrize("flag", ["binary", "tree", "eytz"])
@pytest.mark.parametrize("scheme", ["tpl_nw", "silo", "mvcc", "gacco"])
def test_c1_parity_binary_index(c1, orc, scheme, flag):
    """The paper's binary-search index (CC_FLAG_INDEX_BINARY), the cache-line tree
    (CC_FLAG_INDEX_TREE) and the Eytzinger layout (CC_FLAG_INDEX_EYTZ) give the same
    results as the default direct addressing."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_INDEX_BINARY, CC_FLAG_INDEX_EYTZ, CC_FLAG_INDEX_TREE
    fl = {"binary": CC_FLAG_INDEX_BINARY, "tree": CC_FLAG_INDEX_TREE, "eytz": CC_FLAG_INDEX_EYTZ}[flag]
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 44, T, A)
    keys, ops = orc.ycsb_gen(44, 1024, 1024, 4, 0.5, T, A)
    for lanes in (1, 4):
        db.snapshot(False)
        res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes, flags=fl)
        db.sync()
        orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("lanes", [1, 4])
@pytest.mark.parametrize("scheme", ["tpl_nw", "tpl_wd", "to", "mvcc", "silo", "tictoc"])
def test_c1_parity_latched(c1, orc, scheme, lanes):
    """Exp-7 latched variants: same serializable results."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_LATCHED
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 51, T, A)
    keys, ops = orc.ycsb_gen(51, 1024, 1024, 4, 0.5, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes, flags=CC_FLAG_LATCHED)
    assert db.sync().commits == 1024
    orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    b.free()


@pytest.mark.parametrize("lanes", [1, 4])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_stage_breakdown(c1, orc, scheme, lanes):
    """Exp-6 stage accounting: every attempt is counted, stages are
    non-negative and results are unchanged with the timers on."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_STAGES
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 52, T, A)
    keys, ops = orc.ycsb_gen(52, 1024, 1024, 4, 0.5, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes, flags=CC_FLAG_STAGES)
    st = db.sync()
    orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    sc = list(st.stage_cycles)
    assert sc[6] == st.commits + st.aborts               # attempts
    assert sc[0] > 0 and sc[5] > 0                        # index lookups and row work happened
    if st.aborts == 0:
        assert sc[4] == 0                                 # no abort time without aborts
    if scheme in ("to", "mvcc"):
        assert sc[1] > 0                                  # timestamp allocation
    b.free()


@pytest.mark.parametrize("lanes", [1, 4])
@pytest.mark.parametrize("scheme", ["tpl_nw", "tpl_wd", "to", "silo", "tictoc", "gputx", "gacco"])
def test_event_log_conflict_graph(c1, orc, scheme, lanes):
    """f-4 debug mode: the device event log of a high-contention batch yields an acyclic
    conflict graph, with one commit event per transaction."""
    from paper_2406_10158_b200.gcctb import CC_FLAG_EVENTS
    from paper_2406_10158_b200.verify import check_serializable
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 53, T, A)
    keys, ops = orc.ycsb_gen(53, 1024, 1024, 4, 0.5, T, A)
    db.events_capacity(1 << 22)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=32, lanes=lanes, flags=CC_FLAG_EVENTS)
    st = db.sync()
    orc.check_ycsb(scheme, S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
    ev = db.events()
    assert int((ev["kind"] == 2).sum()) == 1024
    assert int((ev["kind"] == 3).sum()) == st.aborts
    ok, info = check_serializable(ev)
    assert ok, f"cycle {info}"
    b.free()


def test_device_error_is_sticky_across_submits(c1):
    """A device error of an earlier submit is reported by the next cc_sync even when
    later submits (which reset the per-submit control block) succeeded."""
    from paper_2406_10158_b200.gcctb import CCError
    db, _ = c1
    bad = db.import_ycsb(np.array([1, 5000], np.uint32), np.array([0, 0], np.uint8), 2)
    good = db.import_ycsb(np.array([1, 2], np.uint32), np.array([0, 0], np.uint8), 2)
    db.submit(bad, "tictoc")
    db.submit(good, "tictoc")
    with pytest.raises(CCError, match="KEY_NOT_FOUND"):
        db.sync()
    db.submit(good, "tictoc")
    assert db.sync().commits == 1     # cleared after being reported
    bad.free()
    good.free()


def test_import_async_host(c1, orc):
    """CC_SRC_HOST_ASYNC: pinned host batches copied on the copy stream (overlapping queued
    work; a pooled buffer's previous readers finish first) give the oracle's results."""
    import torch
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    for seed in (61, 62, 63):
        keys, ops = orc.ycsb_gen(seed, 1024, 1024, 4, 0.5, T, A)
        pk, po = torch.from_numpy(keys).pin_memory(), torch.from_numpy(ops).pin_memory()
        db.snapshot(False)
        b = db.import_ycsb(pk, po, 4, async_host=True)
        res = db.submit(b, "tictoc", wd=0, bs=32, lanes=4)
        db.sync()
        orc.check_ycsb("tictoc", S0, keys, ops, 4, res.host(db.stream), db.read_table(0))
        b.free()


# Ragged shapes: a single transaction, batch sizes that leave a partial last tile / warp /
# block, K that leaves idle lanes in a 4/8/16-lane tile, K=1.
RAGGED = [(1, 16), (4099, 5), (2053, 16), (777, 1), (33, 3)]


@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("n,K", RAGGED)
def test_ragged_shapes(c1, orc, scheme, n, K):
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(n, K, 0.5, 100 + n + K, T, A)
    keys, ops = orc.ycsb_gen(100 + n + K, 1024, n, K, 0.5, T, A)
    for lanes in [1] + [L for L in (4, 8, 16) if L >= K]:
        db.snapshot(False)
        res = db.submit(b, scheme, wd=0, bs=32 if n > 64 else 1, lanes=lanes)
        st = db.sync()
        assert st.commits == n, (lanes, st.commits)
        h = res.host(db.stream)
        assert int(h["restarts"].astype(np.int64).sum()) == st.aborts
        orc.check_ycsb(scheme, S0, keys, ops, K, h, db.read_table(0))
    b.free()


def test_bad_geometry_is_rejected_before_enqueue(c1):
    """include/gcctb.h: argument / config errors return before anything is enqueued and
    leave the db usable."""
    from paper_2406_10158_b200.gcctb import CCError, STATUS_NAMES
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    for n, K in [(0, 4), (16, 0), (16, 17), ((1 << 21) + 1, 4)]:
        with pytest.raises(CCError) as e:
            db.gen_ycsb(n, K, 0.5, 1, T, A)
        assert STATUS_NAMES[e.value.status] in ("CONFIG", "INVALID_ARG")
    with pytest.raises(CCError) as e:
        db.import_ycsb(np.zeros(0, np.uint32), np.zeros(0, np.uint8), 4)
    assert STATUS_NAMES[e.value.status] == "INVALID_ARG"
    b = db.gen_ycsb(64, 8, 0.5, 1, T, A)
    with pytest.raises(CCError) as e:      # an 8-op transaction does not fit a 4-lane tile
        db.submit(b, "silo", lanes=4)
    assert STATUS_NAMES[e.value.status] == "INVALID_ARG"
    db.snapshot(False)
    db.submit(b, "silo", lanes=8)          # the db is still usable
    assert db.sync().commits == 64
    b.free()


@pytest.mark.parametrize("lanes", [1, 8])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c1_all_writes_extreme_contention(c1, orc, scheme, lanes):
    """W=1, theta=0.99 on the 1,024-row table: every access a write, ~40 % of them on one
    row -- the abort, retry-pacing, hot-first, wait-die intent and TO sequential paths all
    fire; parity must hold and every transaction commits."""
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.99)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(512, 8, 1.0, 29, T, A)
    keys, ops = orc.ycsb_gen(29, 1024, 512, 8, 1.0, T, A)
    db.snapshot(False)
    res = db.submit(b, scheme, wd=0, bs=8, lanes=lanes, watchdog_s=60)
    st = db.sync()
    assert st.commits == 512
    h = res.host(db.stream)
    assert int(h["restarts"].astype(np.int64).sum()) == st.aborts
    orc.check_ycsb(scheme, S0, keys, ops, 8, h, db.read_table(0))
    b.free()


def test_generator_failure_is_reported_at_submit(torch_cuda):
    """an a1 failure (no distinct keys drawable: every threshold 0 puts all the
    Zipf mass on one rank) stays with its batch -- the next submit's a2 reset does not
    erase it -- so the submit executes nothing and cc_sync reports CONFIG; the db is not
    sticky-failed, a valid batch afterwards commits normally."""
    from paper_2406_10158_b200.api import DB
    from paper_2406_10158_b200.gcctb import CCError
    db = DB(0)
    db.load_ycsb(64, 3)
    T0 = np.zeros(64, np.uint64)
    bad = db.gen_ycsb(1, 2, 0.0, 1, T0, 5)
    res = db.submit(bad, "tpl_nw", lanes=1, wd=0, bs=1)
    with pytest.raises(CCError, match="CONFIG"):
        db.sync()
    assert int(res.committed.cpu().sum()) == 0
    bad.free()
    T = inputs.zipf_thresholds(64, 0.5)
    ok = db.gen_ycsb(32, 2, 0.5, 2, T, 5)
    db.submit(ok, "tpl_nw", lanes=1, wd=0, bs=1)
    assert db.sync().commits == 32
    ok.free()
    db.close()


@pytest.mark.parametrize("scheme", SCHEMES)
def test_host_result_buffers(c1, orc, scheme):
    """cc_result in pinned host memory (results to host or device): the
    submit stages them on the device and copies them out on the copy stream; after sync
    they equal a device-buffer run's and pass the oracle check.  Several submits in a row
    exercise the two alternating staging sets."""
    from paper_2406_10158_b200.api import Result
    db, S0 = c1
    T = inputs.zipf_thresholds(1024, 0.8)
    A = inputs.scramble_mult(1024)
    b = db.gen_ycsb(1024, 4, 0.5, 31, T, A)
    keys, ops = orc.ycsb_gen(31, 1024, 1024, 4, 0.5, T, A)
    hs = [Result.alloc_host(1024, 4) for _ in range(3)]
    for h in hs:
        db.snapshot(False)
        db.prepare(b, scheme)
        db.submit(b, scheme, wd=0, bs=8, lanes=16, result=h)
        assert db.sync().commits == 1024
        orc.check_ycsb(scheme, S0, keys, ops, 4, h.host(), db.read_table(0))
        assert int(h.stats[0]) == 1024
    b.free()
