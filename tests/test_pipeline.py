"""Training-data pipeline host side (csrc/pipeline.cu) — no GPU needed.

The plan, replay rows and epoch seed run on the host inside libmoses_gpu (the device only gathers),
so they are checked here bit-exactly against the oracle's pure-Python restatement of data.cpp /
tuner.cpp, over the reference's own test_data.cpp scenarios. The record reader / writer is checked
for the behaviour test_data.cpp pins (round trip, byte-identical rewrite, parse errors naming the
line, missing fields)."""
import json
import os

import numpy as np
import pytest

TOY_DEVICE = {"id": "toy", "peak_gflops": 1000.0, "parallel_units": 16.0, "vector_lanes": 8.0,
              "cache_bytes": 1e6, "measure_overhead_ms": 1.0, "noise_std": 0.05, "repeats": 3}


def toy_task(tid, ideal_tiles):  # test_data.cpp:39-48
    return tid, (1.0, 4.0, ideal_tiles, 3.0)


@pytest.fixture(scope="module")
def ml():
    from paper_2201_05752_b200 import moseslab

    return moseslab


def store(orc, tasks, per_task, seed):
    return orc.generate_dataset(TOY_DEVICE, tasks, orc.default_knob_template(), per_task, seed)


def test_oracle_rng_pins(orc):
    # SplitMix64(0) first draw (test_rng.cpp:14-16) and KeyBuilder == the C++ oracle's FNV
    assert orc.RngStream(0).next_u64() == 0xE220A8397B1DCDAF
    assert orc.key_builder("abc") == orc.fnv_str("abc")
    assert orc.key_builder(7, "gen", "a") != orc.key_builder(7, "gen", "b")


def test_oracle_generate_dataset_matches_direct_measurement(orc):
    # test_data.cpp:54-75,77-89: seq store-global, per-task blocks, records == measure(config)
    recs = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], 25, 7)
    assert len(recs) == 50 and [r["seq"] for r in recs] == list(range(50))
    assert [r["task_id"] for r in recs] == ["a"] * 25 + ["b"] * 25
    again = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], 25, 7)
    assert all(x["values"] == y["values"] and x["throughput_gflops"] == y["throughput_gflops"]
               for x, y in zip(recs, again))
    other = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], 25, 8)
    assert any(x["values"] != y["values"] for x, y in zip(recs, other))
    knobs = orc.default_knob_template()
    for r in recs[:10]:
        idx = 0
        for (_, dom), v in zip(knobs, r["values"]):
            idx = idx * len(dom) + dom.index(v)
        _, thr, lat, wall = orc.measure_configs(TOY_DEVICE, "a", (1.0, 4.0, 6.0, 3.0), knobs, 7, idx, 1)
        assert (thr[0], lat[0], wall[0]) == (r["throughput_gflops"], r["latency_ms"], r["wall_cost_ms"])


def _lib_plan(ml, recs, batch, seed):
    ids = list(dict.fromkeys(r["task_id"] for r in recs))
    return ml.make_ranking_batches([r["task_id"] for r in recs], ids, batch, seed)


def _same_plan(ml_plan, orc_batches):
    assert len(ml_plan) == len(orc_batches)
    for b, (tid, rows) in enumerate(orc_batches):
        t, r = ml_plan.batch(b)
        assert t == tid and r.tolist() == rows, b


@pytest.mark.parametrize("per_task,batch,seed", [(23, 8, 99), (9, 4, 100), (16, 4, 5), (16, 4, 6), (6, 6, 1),
                                                 (40, 512, 3), (33, 2, 11), (700, 64, 12345)])
def test_plan_matches_oracle(orc, ml, per_task, batch, seed):
    recs = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], per_task, 13)
    want, dropped = orc.make_ranking_batches([r["task_id"] for r in recs], batch, seed)
    plan = _lib_plan(ml, recs, batch, seed)
    _same_plan(plan, want)
    assert plan.dropped_singletons == dropped


def test_plan_reference_cases(orc, ml):
    # test_data.cpp:162-181: 23 rows per task by 8 -> [8,8,7] twice, nothing dropped
    recs = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], 23, 11)
    plan = _lib_plan(ml, recs, 8, 99)
    assert plan.dropped_singletons == 0 and len(plan) == 6
    seen = {"a": 0, "b": 0}
    for b in range(len(plan)):
        tid, rows = plan.batch(b)
        assert 2 <= len(rows) <= 8 and all(recs[i]["task_id"] == tid for i in rows)
        seen[tid] += len(rows)
    assert seen == {"a": 23, "b": 23}
    # test_data.cpp:183-192: 9 rows by 4 leaves one singleton
    one = store(orc, [toy_task("a", 6.0)], 9, 12)
    p = _lib_plan(ml, one, 4, 100)
    assert p.dropped_singletons == 1 and p.off[-1] == 8
    # test_data.cpp:194-210: deterministic per seed, differs across seeds
    recs = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], 16, 13)
    p1, p2, p3 = (_lib_plan(ml, recs, 4, s) for s in (5, 5, 6))
    assert np.array_equal(p1.rows, p2.rows) and np.array_equal(p1.task, p2.task)
    assert not (np.array_equal(p1.rows, p3.rows) and np.array_equal(p1.task, p3.task))
    # test_data.cpp:212-222: one batch holds every row of the task
    six = store(orc, [toy_task("a", 6.0)], 6, 14)
    p = _lib_plan(ml, six, 6, 1)
    assert len(p) == 1 and sorted(p.rows.tolist()) == list(range(6))


def test_plan_validation(ml):
    # test_data.cpp:224-232
    with pytest.raises(ml.MosesError) as e:
        ml.make_ranking_batches([0, 0, 0], ["a"], 1, 0)
    assert e.value.code == "invalid-config"
    empty = ml.make_ranking_batches([], ["a"], 4, 0)
    assert len(empty) == 0 and empty.dropped_singletons == 0
    with pytest.raises(ml.MosesError) as e:
        ml.make_ranking_batches([0, 3], ["a"], 4, 0)
    assert e.value.code == "invalid-task"


def test_plan_interleaved_store_and_threads(orc, ml):
    # rows of a task need not be contiguous; >= 65536 records takes the threaded shuffle path
    rng = np.random.default_rng(0)
    ids = ["t%d" % i for i in range(5)]
    tasks = [ids[i] for i in rng.integers(0, 5, 70000)]
    want, dropped = orc.make_ranking_batches(tasks, 512, 77)
    plan = ml.make_ranking_batches(tasks, ids, 512, 77)
    # task indices follow first appearance in the oracle; compare by id
    _same_plan(plan, want)
    assert plan.dropped_singletons == dropped


def test_replay_rows_and_epoch_seed(orc, ml):
    for n, size, seed in [(40, 12, 77), (5, 12, 1), (1000, 256, 9)]:
        assert ml.replay_rows(n, size, seed).tolist() == orc.replay_rows(n, size, seed)
    with pytest.raises(ml.MosesError) as e:
        ml.replay_rows(0, 4, 1)
    assert e.value.code == "empty-dataset"
    with pytest.raises(ml.MosesError) as e:
        ml.replay_rows(4, 0, 1)
    assert e.value.code == "invalid-config"
    for s, ep in [(0, 0), (12345, 3), (2**63 + 5, 17)]:
        assert ml.epoch_seed(s, ep) == orc.epoch_seed(s, ep)


# ---------------------------------------------------------------- record files (data.cpp:67-126)
def _to_store(ml, recs):
    st = ml.RecordStore()
    for r in recs:
        st.append(r["task_id"], r["device_id"], r["values"], r["throughput_gflops"], r["latency_ms"],
                  r["wall_cost_ms"], r["seq"])
    return st


def test_records_roundtrip_byte_identical(orc, ml, tmp_path):
    # test_data.cpp:115-143
    recs = store(orc, [toy_task("a", 6.0), toy_task("b", 9.0)], 12, 5)
    p1, p2 = str(tmp_path / "r1.jsonl"), str(tmp_path / "r2.jsonl")
    _to_store(ml, recs).write(p1)
    back = ml.RecordStore.read(p1)
    ex = back.export()
    assert len(back) == 24 and back.task_ids() == ["a", "b"] and back.device_ids() == ["toy"]
    for i, r in enumerate(recs):
        assert ex["values"][ex["value_off"][i]:ex["value_off"][i + 1]].tolist() == r["values"]
        assert ex["throughput"][i] == r["throughput_gflops"] and ex["wall_cost"][i] == r["wall_cost_ms"]
        assert ex["latency"][i] == r["latency_ms"] and int(ex["seq"][i]) == r["seq"]
    back.write(p2)
    b1, b2 = open(p1, "rb").read(), open(p2, "rb").read()
    assert b1 == b2 and b1.endswith(b"\n")
    # every line is the key-sorted compact JSON object the reference's writer produces
    for line, r in zip(b1.decode().splitlines(), recs):
        want = {k: r[k] for k in ("task_id", "values", "throughput_gflops", "latency_ms", "wall_cost_ms",
                                  "device_id", "seq")}
        assert json.loads(line) == want
        assert line == json.dumps(want, sort_keys=True, separators=(",", ":"))


def test_records_read_foreign_lines(ml, tmp_path):
    # field order, whitespace, escapes, unicode, integral floats, unknown fields, blank lines
    rec = {"task_id": 'weird "quoted" id\té\U0001F600', "values": [8, 64, 0, 1, 256],
           "throughput_gflops": 123.45678901234567, "latency_ms": 0.0078125, "wall_cost_ms": 1.5,
           "device_id": "dev", "seq": 9001}
    p = str(tmp_path / "f.jsonl")
    with open(p, "w") as f:
        f.write(json.dumps(rec) + "\n\n")
        f.write(' { "seq" : 2 , "values":[1.0, 2], "extra": {"x": [null, true]}, "task_id":"b",'
                '"device_id":"dev","throughput_gflops":3,"latency_ms":1e-3,"wall_cost_ms":2E+1 }\n')
    st = ml.RecordStore.read(p)
    ex = st.export()
    assert st.task_ids() == [rec["task_id"], "b"] and len(st) == 2
    assert ex["values"].tolist() == [8, 64, 0, 1, 256, 1, 2] and ex["value_off"].tolist() == [0, 5, 7]
    assert ex["throughput"].tolist() == [rec["throughput_gflops"], 3.0]
    assert ex["latency"].tolist() == [0.0078125, 1e-3] and ex["wall_cost"].tolist() == [1.5, 20.0]
    assert ex["seq"].tolist() == [9001, 2]
    out = str(tmp_path / "g.jsonl")
    st.write(out)
    first = json.loads(open(out).read().splitlines()[0])
    assert first == rec


def test_records_errors(ml, tmp_path):
    # test_data.cpp:108-113,145-160
    p = str(tmp_path / "bad.jsonl")
    good = json.dumps({"task_id": "a", "values": [1], "throughput_gflops": 1.0, "latency_ms": 1.0,
                       "wall_cost_ms": 1.0, "device_id": "d", "seq": 0})
    for body, code, needle in [(good + "\ngarbage\n", "parse-error", "line 2"),
                               ('{"task_id":"a"}\n', "missing-field", "line 1"),
                               (good + "\n" + good + " x\n", "parse-error", "line 2"),
                               (good.replace('"a"', "5") + "\n", "parse-error", "line 1"),
                               (good.replace("[1]", '["x"]') + "\n", "parse-error", "line 1"),
                               ('{"task_id":"a", }\n', "parse-error", "line 1")]:
        with open(p, "w") as f:
            f.write(body)
        with pytest.raises(ml.MosesError) as e:
            ml.RecordStore.read(p)
        assert e.value.code == code and needle in str(e.value), (body, str(e.value))
    with pytest.raises(ml.MosesError) as e:
        ml.RecordStore.read(str(tmp_path / "missing.jsonl"))
    assert e.value.code == "io-error"


@pytest.mark.parametrize("x,want", [(1.0, "1.0"), (1.5, "1.5"), (0.0078125, "0.0078125"), (1e-5, "1e-05"),
                                    (123.45678901234567, "123.45678901234567"), (1e14, "100000000000000.0"),
                                    (1e15, "1e+15"), (-2.5e-7, "-2.5e-07"), (0.0001, "0.0001"), (0.1, "0.1")])
def test_records_number_format(ml, tmp_path, x, want):
    # nlohmann::json's float layout (fixed for -4 < exponent+1 <= 15)
    st = ml.RecordStore()
    st.append("a", "d", [1], x, 1.0, 1.0, 0)
    p = str(tmp_path / "n.jsonl")
    st.write(p)
    line = open(p).read()
    assert '"throughput_gflops":' + want + "," in line, line
    assert ml.RecordStore.read(p).export()["throughput"][0] == x


def test_records_roundtrip_property(ml, tmp_path):
    """Any record (unicode ids with escapes, any finite double, int64 values, u64 seq) survives
    write -> read unchanged, and the writer's lines parse as the same JSON object."""
    hypothesis = pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    path = str(tmp_path / "prop.jsonl")
    # ids cross the C ABI as NUL-terminated UTF-8: no embedded NUL, no lone surrogates
    text = st.text(alphabet=st.characters(blacklist_categories=("Cs",), blacklist_characters="\x00"),
                   min_size=0, max_size=12)
    dbl = st.floats(allow_nan=False, allow_infinity=False, width=64)
    rec = st.tuples(text, text, st.lists(st.integers(-2**63, 2**63 - 1), max_size=6), dbl, dbl, dbl,
                    st.integers(0, 2**64 - 1))

    @settings(max_examples=60, deadline=None)
    @given(st.lists(rec, min_size=1, max_size=5))
    def check(records):
        store = ml.RecordStore()
        for tid, did, vals, thr, lat, wall, seq in records:
            store.append(tid, did, [vals] if vals else np.zeros((1, 0), dtype=np.int64), thr, lat, wall, seq)
        store.write(path)
        back = ml.RecordStore.read(path).export()
        ids = ml.RecordStore.read(path)
        tids, dids = ids.task_ids(), ids.device_ids()
        lines = open(path, encoding="utf-8").read().split("\n")  # not splitlines(): U+0085 is valid in JSON strings
        for i, (tid, did, vals, thr, lat, wall, seq) in enumerate(records):
            assert tids[back["task"][i]] == tid and dids[back["device"][i]] == did
            assert back["values"][back["value_off"][i]:back["value_off"][i + 1]].tolist() == vals
            assert back["throughput"][i] == thr and back["latency"][i] == lat and back["wall_cost"][i] == wall
            assert int(back["seq"][i]) == seq
            obj = json.loads(lines[i])
            assert obj["task_id"] == tid and obj["values"] == vals and obj["seq"] == seq
            assert obj["throughput_gflops"] == thr

    check()


def test_plan_property_vs_oracle(orc, ml):
    """Random stores (task interleavings, batch sizes, seeds): the native plan equals the oracle's
    make_ranking_batches restatement batch for batch."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @settings(max_examples=80, deadline=None)
    @given(st.lists(st.integers(0, 4), max_size=120), st.integers(2, 40), st.integers(0, 2**64 - 1))
    def check(tasks, batch, seed):
        ids = ["task%d" % t for t in range(5)]
        rec = [ids[t] for t in tasks]
        want, dropped = orc.make_ranking_batches(rec, batch, seed)
        plan = ml.make_ranking_batches(rec, ids, batch, seed)
        _same_plan(plan, want)
        assert plan.dropped_singletons == dropped
        got_rows = sorted(plan.rows.tolist())
        assert got_rows == sorted(r for _, rows in want for r in rows)

    check()


def test_records_reader_fuzz(ml, tmp_path):
    """Arbitrary (often malformed) lines never crash the native reader: each file either reads or
    fails with parse-error / missing-field naming a line."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    path = str(tmp_path / "fuzz.jsonl")
    good = ('{"task_id":"a","values":[1,2],"throughput_gflops":1.5,"latency_ms":2,"wall_cost_ms":3,'
            '"device_id":"d","seq":4}')
    pieces = st.sampled_from(['{', '}', '[', ']', '"', ':', ',', '\\', '\\u12', 'true', 'null', '1e400', '-0',
                              '"task_id"', '"values"', '"seq"', ' ', '\t', good, good[:-1], good[1:]])
    line = st.one_of(st.lists(pieces, max_size=12).map("".join), st.text(max_size=40))

    @settings(max_examples=300, deadline=None)
    @given(st.lists(line, min_size=1, max_size=4))
    def check(lines):
        with open(path, "w", encoding="utf-8", errors="surrogatepass") as f:
            f.write("\n".join(lines) + "\n")
        try:
            ml.RecordStore.read(path)
        except ml.MosesError as e:
            assert e.code in ("parse-error", "missing-field"), e
            assert ":line " in str(e)

    check()
