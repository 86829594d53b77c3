# SPDX-License-Identifier: Apache-2.0
"""The C++ drop-in: reference-style callers compiled against <repo>/include's
gridmath/*.hpp headers (the reference's include paths) and linked with
libgridmath_b200.so (tests/cpp/Makefile).

* dropin_callsites: one hidden FC layer step in the Trainer's call order,
  recorded and replayed, plus the rest of the reference's public Session
  surface and the out-of-path entry points;
* dropin_dnn: the reference's UNMODIFIED dnn.cpp (Trainer) -- built where
  /root/reference exists, the binary travels to the GPU box."""
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CPP = os.path.join(ROOT, "tests", "cpp")
BUILD = os.path.join(CPP, "_build")


def _make():
    subprocess.check_call(["make", "-s", "-C", CPP], stdout=subprocess.DEVNULL)


def test_dropin_headers_compile_and_link():
    """CPU: the reference-style call sites (and, with the reference sources
    present, its unchanged dnn.cpp) compile against the drop-in headers and
    every symbol resolves in libgridmath_b200.so."""
    if not shutil.which("g++"):
        pytest.skip("no g++")
    _make()
    exe = os.path.join(BUILD, "dropin_callsites")
    assert os.path.exists(exe)
    bins = [exe]
    if os.path.exists("/root/reference/proj/src/dnn.cpp"):
        assert os.path.exists(os.path.join(BUILD, "dropin_dnn"))
        bins.append(os.path.join(BUILD, "dropin_dnn"))
    for b in bins:
        out = subprocess.run(["ldd", "-r", b], capture_output=True, text=True)
        assert "undefined symbol" not in out.stdout + out.stderr, out.stdout + out.stderr
        assert "libgridmath_b200.so" in out.stdout


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_dropin_callsites_fc_step_matches_numpy(tmp_path):
    _make()
    out = os.path.join(tmp_path, "fc.bin")
    r = subprocess.run([os.path.join(BUILD, "dropin_callsites"), out], capture_output=True, text=True, timeout=500)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout + r.stderr
    v = np.fromfile(out, dtype=np.float64)
    batch, fi, fo, lr = 256, 384, 192, 0.05
    shapes = [(batch, fi), (fi, fo), (1, fo), (batch, fo)] + [(batch, fo), (batch, fo), (fi, fo), (1, fo),
                                                              (batch, fi), (fi, fo), (1, fo)] * 2
    arrs, o = [], 0
    for sh in shapes:
        n = sh[0] * sh[1]
        arrs.append(v[o:o + n].reshape(sh))
        o += n
    assert o == v.size
    x, w, b, g = arrs[:4]
    for step in range(2):
        z, act, dw, db, dx, w1, b1 = arrs[4 + 7 * step: 11 + 7 * step]
        assert _rel(z, x @ w + b) <= 1e-5
        assert np.array_equal(act, np.where(z > 0, z, 0.0))
        delta = np.where(z > 0, g, 0.0)  # reluGrad on the device's own pre-activation
        assert _rel(dw, x.T @ delta) <= 1e-5
        assert _rel(db, delta.sum(axis=0, keepdims=True)) <= 1e-5
        assert _rel(dx, delta @ w.T) <= 1e-5
        assert np.array_equal(w1, _f32(_f32(w) - _f32(lr * dw)).astype(np.float64)) or _rel(w1, w - lr * dw) <= 1e-6
        assert _rel(b1, b - lr * db) <= 1e-6
        w, b = w1, b1


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_reference_dnn_trainer_runs_on_the_dropin(tmp_path):
    exe = os.path.join(BUILD, "dropin_dnn")
    if not os.path.exists(exe):
        pytest.skip("dropin_dnn not built (needs the reference sources at build time)")
    out = os.path.join(tmp_path, "dnn.bin")
    r = subprocess.run([exe, out], capture_output=True, text=True, timeout=500)
    assert r.returncode == 0 and "DROPIN_DNN OK" in r.stdout, r.stdout + r.stderr
    raw = open(out, "rb").read()
    n, dim, classes = np.frombuffer(raw[:12], dtype=np.uint32)
    o = 12
    feats = np.frombuffer(raw[o:o + 4 * n * dim], dtype=np.float32).reshape(n, dim).astype(np.float64)
    o += 4 * n * dim
    params = []
    for _ in range(4):
        cnt = int(np.frombuffer(raw[o:o + 8], dtype=np.uint64)[0])
        o += 8
        params.append(np.frombuffer(raw[o:o + 8 * cnt], dtype=np.float64).copy())
        o += 8 * cnt
    pred = np.frombuffer(raw[o:o + 4 * n], dtype=np.uint32)
    half = np.frombuffer(raw[o + 4 * n:o + 8 * n], dtype=np.uint32)
    hidden = params[1].size
    w0 = params[0].reshape(dim, hidden)
    w1 = params[2].reshape(hidden, classes)
    h = np.maximum(feats @ w0 + params[1], 0.0)
    logits = h @ w1 + params[3]
    want = logits.argmax(axis=1)
    top2 = np.sort(logits, axis=1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 1e-4 * np.abs(top2[:, 1]).clip(1.0)
    assert np.array_equal(pred[clear], want[clear])
    # mixed Half weights: the same decisions except on near-ties
    assert (half[clear] == want[clear]).mean() >= 0.97
