# SPDX-License-Identifier: Apache-2.0
"""Pipeline record / replay (reference Session::beginRecord / endRecord /
replay, session.cpp:385-409; recordable ops session.cpp:16-30), on the
device path: a recorded FC train step replayed K times equals the same step
issued eagerly K+1 times, bit-for-bit, with the same matrix versions."""
import numpy as np
import pytest

from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu


def build(s, p, S=G.Precision.Single, batch=192, fin=256, fout=160):
    grp = list(range(p))
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


@pytest.mark.parametrize("p,prec,shape", [
    (1, G.Precision.Single, (192, 256, 160)),
    (4, G.Precision.Single, (192, 256, 160)),
    # bf16: replay runs gemm -> biasAdd -> relu as one GEMM with the fused
    # epilogue; eager runs the three ops. Bitwise equal either way.
    (1, G.Precision.BF16, (192, 256, 160)),
    (4, G.Precision.BF16, (192, 256, 160)),
    (2, G.Precision.BF16, (200, 96, 136)),
    (3, G.Precision.BF16, (515, 320, 1000)),
])
def test_replay_equals_eager(p, prec, shape):
    k = 3
    batch, fin, fout = shape
    with G.Session(workers=p) as s:
        m = build(s, p, prec, batch, fin, fout)
        pid = s.beginRecord()
        step(s, m)
        s.endRecord()
        for _ in range(k):
            s.replay(pid)
        s.verifyMetadataConsistency()
        got = snapshot(s, m)
    with G.Session(workers=p) as s:
        m = build(s, p, prec, batch, fin, fout)
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


def test_replay_fuses_bias_relu_into_the_gemm():
    # The bf16 step's replay launches four kernels fewer than the eager step:
    # biasAdd and relu ride in the forward GEMM's epilogue, and the two
    # setConst(0) before addRowColSum become the sums' zero start. Single only
    # takes the second peephole.
    counts = {}
    for prec in (G.Precision.BF16, G.Precision.Single):
        with G.Session(workers=1) as s:
            m = build(s, 1, prec)
            pid = s.beginRecord()
            step(s, m)
            s.endRecord()
            s.synchronize()
            n0 = G.kernel_launches()
            step(s, m)
            s.synchronize()
            n1 = G.kernel_launches()
            s.replay(pid)
            n2 = G.kernel_launches()
            counts[prec] = (n1 - n0, n2 - n1)
    eager, replayed = counts[G.Precision.BF16]
    assert replayed == eager - 4, counts
    eager, replayed = counts[G.Precision.Single]
    assert replayed == eager - 2, counts


def test_fused_epilogue_not_used_when_bias_needs_a_transfer():
    # Z row-block over 2 workers, bias col-block and not replicated: each
    # worker's Z tile needs bias columns the other owns, so replay keeps the
    # three ops (and still matches eager).
    def run(record):
        with G.Session(workers=2) as s:
            P = G.Precision.BF16
            grp = [0, 1]
            X = s.createMatrix(64, 96, P, G.makeRowBlockLayout(64, 96, grp))
            W = s.createMatrix(96, 80, P, G.makeColBlockLayout(96, 80, grp))
            B = s.createMatrix(1, 80, P, G.makeColBlockLayout(1, 80, grp))
            Z = s.createMatrix(64, 80, P, G.makeRowBlockLayout(64, 80, grp))
            A = s.createMatrix(64, 80, P, G.makeRowBlockLayout(64, 80, grp))
            s.fillUniform(X, 1)
            s.fillUniform(W, 2)
            s.fillUniform(B, 3)
            def fwd():
                G.gemm(s, X, W, Z, 1.0, 0.0)
                G.biasAdd(s, Z, B)
                G.relu(s, Z, A)
            if record:
                pid = s.beginRecord()
                fwd()
                s.endRecord()
                s.replay(pid)
            else:
                fwd()
                fwd()
            return s.getDataRaw(Z), s.getDataRaw(A), Z.version(), A.version()
    got, want = run(True), run(False)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g), np.asarray(w))


@pytest.mark.parametrize("p,batch,fin,fout", [(2, 128, 192, 256), (3, 100, 64, 264)])
def test_fused_epilogue_on_column_blocks(p, batch, fin, fout):
    # Z / act / bias column blocks with the same split: every worker holds the
    # bias columns of its Z tile, so each worker's GEMM carries the epilogue.
    def run(record):
        with G.Session(workers=p) as s:
            P = G.Precision.BF16
            grp = list(range(p))
            X = s.createMatrix(batch, fin, P, G.makeSingleTileLayout(batch, fin, 0))
            W = s.createMatrix(fin, fout, P, G.makeColBlockLayout(fin, fout, grp))
            B = s.createMatrix(1, fout, P, G.makeColBlockLayout(1, fout, grp))
            Z = s.createMatrix(batch, fout, P, G.makeColBlockLayout(batch, fout, grp))
            A = s.createMatrix(batch, fout, P, G.makeColBlockLayout(batch, fout, grp))
            s.fillUniform(X, 5)
            s.fillUniform(W, 6, -0.2, 0.2)
            s.fillUniform(B, 7, -0.3, 0.3)

            def fwd():
                G.gemm(s, X, W, Z, 1.0, 0.0)
                G.biasAdd(s, Z, B)
                G.relu(s, Z, A)
            s.synchronize()
            n0 = G.kernel_launches()
            if record:
                pid = s.beginRecord()
                fwd()
                s.endRecord()
                s.synchronize()
                n0 = G.kernel_launches()
                s.replay(pid)
            else:
                fwd()
                s.synchronize()
                n0 = G.kernel_launches()
                fwd()
            s.synchronize()
            n = G.kernel_launches() - n0
            return [s.getDataRaw(Z), s.getDataRaw(A), Z.version(), A.version()], n
    (got, n_rep), (want, n_eager) = run(True), run(False)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g), np.asarray(w))
    assert n_rep == n_eager - 2 * p, (n_rep, n_eager)
    a = got[1].view(np.uint16)
    assert (a != 0).any() and not (a & 0x8000).any()  # relu output: non-trivial, no negatives


@pytest.mark.parametrize("p,prec", [(1, G.Precision.BF16), (1, G.Precision.Single), (4, G.Precision.BF16),
                                    (2, G.Precision.Single)])
def test_graph_replay_matches_op_by_op(p, prec):
    # Replays after the first are captured into one CUDA graph (executable
    # updated in place); a new batch is written eagerly between replays, as
    # the bench and the reference Trainer do. Same bits and versions as
    # replays issued op by op.
    k = 5

    def run(graph):
        with G.Session(workers=p) as s:
            s.setGraphReplay(graph)
            m = build(s, p, prec)
            pid = s.beginRecord()
            step(s, m)
            s.endRecord()
            for i in range(k):
                s.fillUniform(m["X"], 100 + i)
                s.replay(pid, sync=(i % 2 == 1))
            s.synchronize()
            s.verifyMetadataConsistency()
            return snapshot(s, m), s.graphStats()

    got, gs = run(True)
    want, off = run(False)
    assert off["launches"] == 0
    assert gs["launches"] == k - 1, gs
    assert 1 <= gs["instantiations"] <= 2, gs
    assert gs["nodes"] > 0
    for name in got:
        assert got[name][1] == want[name][1], name
        assert np.array_equal(got[name][0], want[name][0]), name


def test_graph_replay_keeps_kernel_timing():
    # The per-GEMM timing window rides inside the graph as event-record nodes.
    with G.Session(workers=1) as s:
        s.setGraphReplay(True)
        m = build(s, 1, G.Precision.BF16, 1024, 2048, 1024)
        pid = s.beginRecord()
        step(s, m)
        s.endRecord()
        s.replay(pid)
        s.timerStart()
        for _ in range(3):
            s.replay(pid, sync=False)
        ms = s.timerStop()
        (tot, cnt), = s.timerKernelMs()
        assert s.graphStats()["launches"] == 3
        assert ms > 0 and cnt == 9 and 0 < tot < ms * 1.01, (ms, tot, cnt)


def test_op_timeline_marks_every_replayed_op():
    with G.Session(workers=2) as s:
        m = build(s, 2)
        pid = s.beginRecord()
        step(s, m)
        s.endRecord()
        s.setOpTimeline(True)
        s.replay(pid)
        tl = s.opTimeline()
        # 13 recorded ops; setConst x2 + addRowColSum replay as one mark (zero-sums peephole)
        assert tl[0][0] == "start" and len(tl) == 1 + 11, tl
        assert any(lab == "setConst+setConst+addRowColSum" for lab, _, _ in tl), tl
        comp = [c for _, c, _ in tl]
        assert comp == sorted(comp) and comp[-1] > 0, tl
        assert [lab for lab, _, _ in tl[1:4]] == ["gemm", "binary", "unary"], tl


def test_zero_sums_peephole_matches_setconst_then_sums():
    # setConst(R, 0), setConst(C, 0), addRowColSum(X, R, C) replayed with the
    # peephole (sums start from zero, no setConst kernels) == the three ops
    # run one by one, bit-for-bit and version-for-version, also when R and C
    # held other values before and alpha is negative (a -0 product stays +0).
    def run(fuse, p, prec):
        with G.Session(workers=p) as s:
            m = build(s, p, prec)
            G.setConst(s, m["R"], 3.5)
            G.setConst(s, m["DB"], -2.0)
            pid = s.beginRecord()
            G.setConst(s, m["R"], 0.0)
            G.setConst(s, m["DB"], 0.0)
            G.addRowColSum(s, m["D"], m["R"], m["DB"], -0.75, True)
            s.endRecord()
            G.setConst(s, m["R"], 7.0)
            if not fuse:
                G.setConst(s, m["R"], 0.0)
                G.setConst(s, m["DB"], 0.0)
                G.addRowColSum(s, m["D"], m["R"], m["DB"], -0.75, True)
            else:
                s.replay(pid)
            return {k: (s.getDataRaw(m[k]), m[k].version()) for k in ("R", "DB")}
    for p, prec in ((1, G.Precision.BF16), (2, G.Precision.Single), (3, G.Precision.BF16)):
        got, want = run(True, p, prec), run(False, p, prec)
        for k in got:
            assert got[k][1] == want[k][1], (k, p, prec)
            assert np.array_equal(got[k][0], want[k][0]), (k, p, prec)
