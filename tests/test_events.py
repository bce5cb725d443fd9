"""Columnar event ingest + device feature extraction (SPEC.md:32-70,
113-121).  CPU: read_trace / validate_event semantics and the ESCOL1 round trip; GPU:
es_events_extract against a numpy restatement of extract_features."""
import json

import numpy as np
import pytest

from paper_2506_02007_b200 import events as ev


def write_jsonl(path, recs, raw_lines=None):
    with open(path, "w") as fh:
        for r in recs:
            fh.write(json.dumps(r) + "\n")
        for line in raw_lines or []:
            fh.write(line + "\n")


NCCL = {"layer": "Nccl", "kind": "ncclAllReduce", "ts_start": 10, "duration_ns": 500, "pid": 1, "tid": 1,
        "attrs": {"message_bytes": 4096}}


def random_records(n, seed=0):
    rng = np.random.default_rng(seed)
    recs = []
    for i in range(n):
        lay = ["Cuda", "Python", "Torch", "Nccl", "GpuSample"][rng.integers(0, 5)]
        r = {"layer": lay, "kind": f"k{rng.integers(0, 7)}", "ts_start": int(1 + i * 1000), "pid": 7, "tid": int(i % 3),
             "duration_ns": 0 if lay == "GpuSample" else int(rng.integers(0, 10 ** 9)), "attrs": {}}
        if lay == "Nccl":
            r["attrs"]["message_bytes"] = int(rng.integers(0, 1 << 30))
        if lay == "GpuSample":
            r["attrs"] = {"util_pct": float(rng.uniform(0, 100)), "mem_used_mb": float(rng.uniform(0, 80000)),
                          "temp_c": float(rng.uniform(20, 90)), "power_w": 300.0}
            r["device"] = int(rng.integers(0, 8))
        recs.append(r)
    return recs


def features_ref(cols, layer):
    """extract_features default feature sets, restated."""
    L = ev.LAYERS[layer]
    sel = np.nonzero(cols.layer == L)[0]
    if layer == "GpuSample":
        X = np.stack([cols.attrs["util_pct"][sel], cols.attrs["mem_used_mb"][sel], cols.attrs["temp_c"][sel]], 1)
    elif layer == "Nccl":
        X = np.stack([np.log10(cols.duration_ns[sel] + 1.0), np.log10(cols.attrs["message_bytes"][sel] + 1.0)], 1)
    else:
        X = np.log10(cols.duration_ns[sel] + 1.0)[:, None]
    return X, sel


# ------------------------------------------------------------------ CPU
def test_read_trace_examples(tmp_path):
    p = tmp_path / "t.jsonl"
    write_jsonl(p, [])
    assert len(ev.read_trace_jsonl(str(p))) == 0
    write_jsonl(p, [NCCL, dict(NCCL, ts_start=20)])
    c = ev.read_trace_jsonl(str(p))
    assert len(c) == 2 and list(c.ts_start) == [10, 20]
    write_jsonl(p, [NCCL], ["{not json"])
    with pytest.raises(Exception) as e:
        ev.read_trace_jsonl(str(p))
    assert e.value.name == "ParseError" and "line 2" in str(e.value)
    for bad, name in ((dict(NCCL, duration_ns=-1), "RangeViolation"),
                      ({"layer": "GpuSample", "kind": "gpu_sample", "ts_start": 5, "duration_ns": 0, "pid": 1,
                        "tid": 1, "attrs": {"util_pct": 250, "mem_used_mb": 1, "temp_c": 40}}, "RangeViolation"),
                      (dict(NCCL, layer="Disk"), "UnknownLayer"), (dict(NCCL, attrs={}), "MissingField")):
        write_jsonl(p, [bad])
        with pytest.raises(Exception) as e:
            ev.read_trace_jsonl(str(p))
        assert e.value.name == name


def test_columnar_round_trip(tmp_path):
    recs = random_records(1000)
    a = ev.from_records(recs)
    ev.write_columnar(a, str(tmp_path / "e.escol"))
    b = ev.read_columnar(str(tmp_path / "e.escol"))
    assert len(b) == 1000 and b.kinds == a.kinds
    for f in ("layer", "kind", "ts_start", "duration_ns", "pid", "tid", "device"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    for k in ev.ATTRS:
        assert np.array_equal(a.attrs[k], b.attrs[k], equal_nan=True), k
    ev.write_columnar(ev.from_records([]), str(tmp_path / "z.escol"))
    assert len(ev.read_columnar(str(tmp_path / "z.escol"))) == 0


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_extract_examples(es):
    c = ev.from_records([dict(NCCL, duration_ns=999, attrs={"message_bytes": 9})])
    ds, idx = es.extract_features(c, "Nccl")
    assert np.array_equal(ds.read_rows(), np.array([[3.0, 1.0]])) and list(idx) == [0]
    g = {"layer": "GpuSample", "kind": "gpu_sample", "ts_start": 5, "duration_ns": 0, "pid": 1, "tid": 1,
         "attrs": {"util_pct": 50, "mem_used_mb": 1024, "temp_c": 60}}
    ds, idx = es.extract_features(ev.from_records([NCCL, g]), "GpuSample")
    assert np.array_equal(ds.read_rows(), np.array([[50.0, 1024.0, 60.0]])) and list(idx) == [1]


@pytest.mark.gpu
@pytest.mark.parametrize("layer", ["Cuda", "Python", "Torch", "Nccl", "GpuSample"])
def test_extract_parity(es, tmp_path, layer):
    cols = ev.from_records(random_records(20000, seed=3))
    ev.write_columnar(cols, str(tmp_path / "e.escol"))
    cols = ev.read_columnar(str(tmp_path / "e.escol"))
    ds, idx = es.extract_features(cols, layer)
    X, sel = features_ref(cols, layer)
    assert np.array_equal(idx, sel)
    np.testing.assert_allclose(ds.read_rows(), X, rtol=1e-15, atol=0)


@pytest.mark.gpu
def test_extract_validation_on_device(es):
    recs = random_records(500, seed=1)
    c = ev.from_records(recs)
    c.duration_ns[137] = -1
    with pytest.raises(es.EventscopeError) as e:
        es.extract_features(c, "Cuda")
    assert e.value.name == "RangeViolation" and "event 137" in str(e.value)
    c = ev.from_records(recs)
    nccl = int(np.nonzero(c.layer == 3)[0][0])
    c.attrs["message_bytes"][nccl] = np.nan
    with pytest.raises(es.EventscopeError) as e:
        es.extract_features(c, "Cuda")
    assert e.value.name == "MissingField"
    only = ev.from_records([NCCL])
    with pytest.raises(es.EventscopeError) as e:
        es.extract_features(only, "GpuSample")
    assert e.value.name == "EmptyLayer"


@pytest.mark.gpu
def test_columnar_to_pipeline(es, tmp_path):
    """ESCOL1 file -> device features -> run_pipeline, equal to run_pipeline on the host matrix."""
    cols = ev.from_records(random_records(30000, seed=9))
    ev.write_columnar(cols, str(tmp_path / "e.escol"))
    ds, idx = es.extract_features(ev.read_columnar(str(tmp_path / "e.escol")), "Nccl")
    X, _ = features_ref(cols, "Nccl")
    a = es.run_pipeline(ds, 3, quantile_q=0.02, seed=1)
    b = es.run_pipeline(X, 3, quantile_q=0.02, seed=1)
    assert np.array_equal(a.report.flags, b.report.flags)
    np.testing.assert_allclose(a.model.means, b.model.means, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_extract_permutation_and_standardization(es):
    """extract_features is order preserving (permuting events permutes rows)
    and the train-split z-scoring of run_pipeline gives columns with |mean| < 1e-9 and stddev
    within 1e-9 of 1 (FeatureMatrix invariant); x * sigma + m recovers the raw
    features within 1e-9."""
    recs = random_records(6000, seed=12)
    cols = ev.from_records(recs)
    ds, idx = es.extract_features(cols, "Nccl")
    X = ds.read_rows()
    perm = np.random.default_rng(1).permutation(len(recs))
    ds2, idx2 = es.extract_features(ev.from_records([recs[i] for i in perm]), "Nccl")
    X2 = ds2.read_rows()
    pos = {e: r for r, e in enumerate(idx)}
    assert np.array_equal(X2, X[[pos[perm[e]] for e in idx2]])
    r = es.run_pipeline(ds, 3, quantile_q=0.02, seed=0)
    ntr = r.n_train
    Z = (X[:ntr] - r.mean) / r.scale
    assert np.all(np.abs(Z.mean(0)) < 1e-9) and np.all(np.abs(Z.std(0) - 1.0) < 1e-9)
    assert np.allclose(Z * r.scale + r.mean, X[:ntr], rtol=0, atol=1e-9)
