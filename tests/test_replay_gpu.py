# SPDX-License-Identifier: Apache-2.0
"""Pipeline record / replay (reference Session::beginRecord / endRecord /
replay, session.cpp:385-409; recordable ops session.cpp:16-30), on the
device path: a recorded FC train step replayed K times equals the same step
issued eagerly K+1 times, bit-for-bit, with the same matrix versions."""
import numpy as np
import pytest

from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu


def build(s, p):
    grp = list(range(p))
    S = G.Precision.Single
    batch, fin, fout = 192, 256, 160
    m = dict(
        X=s.createMatrix(batch, fin, S, G.makeRowBlockLayout(batch, fin, grp)),
        W=s.createMatrix(fin, fout, S, G.makeColBlockLayout(fin, fout, grp)),
        B=s.createMatrix(1, fout, S, G.makeColBlockLayout(1, fout, grp)),
        Z=s.createMatrix(batch, fout, S, G.makeRowBlockLayout(batch, fout, grp)),
        A=s.createMatrix(batch, fout, S, G.makeRowBlockLayout(batch, fout, grp)),
        D=s.createMatrix(batch, fout, S, G.makeRowBlockLayout(batch, fout, grp)),
        DW=s.createMatrix(fin, fout, S, G.makeColBlockLayout(fin, fout, grp)),
        DB=s.createMatrix(1, fout, S, G.makeColBlockLayout(1, fout, grp)),
        R=s.createMatrix(batch, 1, S, G.makeRowBlockLayout(batch, 1, grp)),
        DX=s.createMatrix(batch, fin, S, G.makeRowBlockLayout(batch, fin, grp)),
    )
    s.fillUniform(m["X"], 1)
    s.fillUniform(m["W"], 2, -0.06, 0.06)
    s.fillUniform(m["B"], 3, -0.1, 0.1)
    s.fillUniform(m["D"], 4)
    s.replicateSync(m["W"])
    s.replicateSync(m["B"])
    return m


def step(s, m, lr=0.01):
    G.gemm(s, m["X"], m["W"], m["Z"], 1.0, 0.0)
    G.biasAdd(s, m["Z"], m["B"])
    G.relu(s, m["Z"], m["A"])
    G.reluGrad(s, m["Z"], m["D"])
    G.gemm(s, m["X"], m["D"], m["DW"], 1.0, 0.0, True, False)
    G.setConst(s, m["R"], 0.0)
    G.setConst(s, m["DB"], 0.0)
    G.addRowColSum(s, m["D"], m["R"], m["DB"], 1.0, True)
    G.gemm(s, m["D"], m["W"], m["DX"], 1.0, 0.0, False, True)
    G.axpy(s, -lr, m["DW"], m["W"])
    G.axpy(s, -lr, m["DB"], m["B"])
    s.replicateAsync(m["W"])
    s.replicateAsync(m["B"])


def snapshot(s, m):
    return {k: (s.getDataRaw(v), v.version()) for k, v in m.items()}


@pytest.mark.parametrize("p", [1, 4])
def test_replay_equals_eager(p):
    k = 3
    with G.Session(workers=p) as s:
        m = build(s, p)
        pid = s.beginRecord()
        step(s, m)
        s.endRecord()
        for _ in range(k):
            s.replay(pid)
        s.verifyMetadataConsistency()
        got = snapshot(s, m)
    with G.Session(workers=p) as s:
        m = build(s, p)
        for _ in range(k + 1):
            step(s, m)
        want = snapshot(s, m)
    for name in got:
        assert got[name][1] == want[name][1], name
        assert np.array_equal(got[name][0], want[name][0]), name


def test_async_replay_then_sync():
    with G.Session(workers=2) as s:
        m = build(s, 2)
        pid = s.beginRecord()
        step(s, m)
        s.endRecord()
        v = m["W"].version()
        s.replay(pid, sync=False)
        s.replay(pid, sync=False)
        s.synchronize()
        assert m["W"].version() == v + 2
        s.verifyMetadataConsistency()


def test_recording_errors_like_reference():
    with G.Session(workers=2) as s:
        m = build(s, 2)
        with pytest.raises(G.GmError, match="no open recording"):
            s.endRecord()
        with pytest.raises(G.GmError, match="unknown or unfinished pipeline 7"):
            s.replay(7)
        pid = s.beginRecord()
        with pytest.raises(G.GmError, match="already open"):
            s.beginRecord()
        with pytest.raises(G.GmError, match="not recordable"):
            s.createMatrix(4, 4, G.Precision.Single, G.makeSingleTileLayout(4, 4, 0))
        with pytest.raises(G.GmError, match="not recordable"):
            s.getDataRaw(m["X"])
        with pytest.raises(G.GmError, match="not recordable"):
            s.reshape(m["X"], G.makeColBlockLayout(192, 256, [0, 1]))
        with pytest.raises(G.GmError, match="recording still open"):
            s.replay(pid)
        G.setConst(s, m["R"], 2.5)
        s.endRecord()
        G.setConst(s, m["R"], 0.0)
        s.replay(pid)
        assert np.all(s.getDataRaw(m["R"]) == np.float32(2.5))
