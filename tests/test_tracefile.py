"""Trace artifacts (tracefile.py): byte compatibility with files the reference
itself wrote (tests/golden/make_golden.py trace_fixture), round trips, and the
reference's validation errors."""

import json
import os
import shutil

import numpy as np
import pytest

from paper_2508_18413_b200 import tracefile as tf

G = os.path.join(os.path.dirname(__file__), "golden")


def test_reads_the_references_file_bit_exact():
    arr, hdr = tf.read_trace(os.path.join(G, "trace_ref.bin"))
    want = np.load(os.path.join(G, "trace_ref_array.npy"))
    assert arr.shape == (2, 5, 3) and arr.tobytes() == want.tobytes()
    assert hdr["sampler"] == "hmc" and hdr["seed"] == 123 and hdr["config"]["L"] == 8


def test_writes_byte_identical_files(tmp_path):
    want = np.load(os.path.join(G, "trace_ref_array.npy"))
    p = tmp_path / "t.bin"
    tf.write_trace(p, want, "hmc", 123, {"eps": 0.5, "L": 8, "method": "quasi-deer"})
    for suffix in ("", ".json"):
        with open(str(p) + suffix, "rb") as a, open(os.path.join(G, "trace_ref.bin" + suffix), "rb") as b:
            assert a.read() == b.read()
    tf.export_csv(tmp_path / "t.csv", want)
    with open(tmp_path / "t.csv", "rb") as a, open(os.path.join(G, "trace_ref.csv"), "rb") as b:
        assert a.read() == b.read()


def test_two_dim_trace_and_torch_tensor(tmp_path):
    torch = pytest.importorskip("torch")
    x = torch.arange(12, dtype=torch.float32).reshape(6, 2)
    hdr = tf.write_trace(tmp_path / "x.bin", x, "mala", 0)
    arr, h2 = tf.read_trace(tmp_path / "x.bin")
    assert hdr == h2 and arr.shape == (1, 6, 2) and np.array_equal(arr[0], x.double().numpy())


def test_validation_errors(tmp_path):
    src = os.path.join(G, "trace_ref.bin")
    p = str(tmp_path / "t.bin")
    shutil.copy(src, p)
    with pytest.raises(tf.TraceFormatError, match="missing sidecar"):
        tf.read_trace(p)
    shutil.copy(src + ".json", p + ".json")
    with open(p, "ab") as fh:  # one extra byte
        fh.write(b"\0")
    with pytest.raises(tf.TraceFormatError, match="payload is"):
        tf.read_trace(p)
    shutil.copy(src, p)
    hdr = json.load(open(p + ".json"))
    for bad, msg in ((dict(hdr, schema_version=2), "schema_version"), (dict(hdr, dtype="f32"), "encoding"),
                     ({k: v for k, v in hdr.items() if k != "D"}, "lacks required field 'D'")):
        json.dump(bad, open(p + ".json", "w"))
        with pytest.raises(tf.TraceFormatError, match=msg):
            tf.read_trace(p)
    open(p + ".json", "w").write("{not json")
    with pytest.raises(tf.TraceFormatError, match="unparseable"):
        tf.read_trace(p)
    with pytest.raises(tf.TraceFormatError, match="expected a"):
        tf.write_trace(p, np.zeros(3), "x", 0)
