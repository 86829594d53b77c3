# SPDX-License-Identifier: Apache-2.0
"""Asynchronous, chunked host<->device streaming of local tiles
(gm_matrix_set/get_local_packed_async): a GEMM that starts on upload row
chunks as they land and a download that drains behind the GEMM's row chunks
must give exactly the results of the synchronous path, across repeated steps
(WAR/RAW ordering of the side streams), with peers pulling a tile that is
still streaming in, and with other ops joining a pending upload."""
import numpy as np
import pytest

import oracle as O
from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu


def packed(s, m):
    return np.zeros(s.localBytes(m), dtype=np.uint8)


def run(p, grid, steps, use_async, n=1024, chunk=48 * 1024):
    outs = []
    with G.Session(workers=p) as s:
        lay = G.makeGridLayout(n, n, grid[0], grid[1], G.makeWorkerGroup(p))
        A = s.createMatrix(n, n, G.Precision.BF16, lay)
        B = s.createMatrix(n, n, G.Precision.BF16, lay)
        C = s.createMatrix(n, n, G.Precision.BF16, lay)
        hosts = []
        for i in range(steps):
            s.fillUniform(A, 10 + i)
            s.fillUniform(B, 50 + i)
            ha, hb = packed(s, A), packed(s, B)
            s.getLocalPacked(A, ha.ctypes.data, ha.nbytes)
            s.getLocalPacked(B, hb.ctypes.data, hb.nbytes)
            hosts.append((ha, hb))
        s.synchronize()
        for ha, hb in hosts:
            hc = packed(s, C)
            if use_async:
                s.setLocalPackedAsync(B, hb.ctypes.data, hb.nbytes, chunk)
                s.setLocalPackedAsync(A, ha.ctypes.data, ha.nbytes, chunk)
                s.gemmAsync(A, B, C)
                s.getLocalPackedAsync(C, hc.ctypes.data, hc.nbytes)
            else:
                s.setLocalPacked(B, hb.ctypes.data, hb.nbytes)
                s.setLocalPacked(A, ha.ctypes.data, ha.nbytes)
                s.gemmAsync(A, B, C)
                s.getLocalPacked(C, hc.ctypes.data, hc.nbytes)
            outs.append(hc)
        s.synchronize()
        ver = C.version()
    return outs, ver


@pytest.mark.parametrize("p,grid", [(1, (1, 1)), (2, (1, 2)), (4, (2, 2))])
def test_async_stream_equals_sync(p, grid):
    got, v1 = run(p, grid, 3, True)
    want, v2 = run(p, grid, 3, False)
    assert v1 == v2
    for i, (g, w) in enumerate(zip(got, want)):
        assert np.array_equal(g, w), i
    assert not np.array_equal(got[0], got[1])  # each step saw its own inputs


def test_async_gemm_matches_oracle():
    n = 768
    with G.Session(workers=1) as s:
        one = G.makeSingleTileLayout(n, n, 0)
        A = s.createMatrix(n, n, G.Precision.BF16, one)
        B = s.createMatrix(n, n, G.Precision.BF16, one)
        C = s.createMatrix(n, n, G.Precision.Single, one)
        a = O.fill_uniform(n, n, 3, 1).reshape(n, n)
        b = O.fill_uniform(n, n, 3, 2).reshape(n, n)
        c = np.zeros((n, n), np.float32)
        s.setLocalPackedAsync(B, b.ctypes.data, b.nbytes, 32 * 1024)
        s.setLocalPackedAsync(A, a.ctypes.data, a.nbytes, 32 * 1024)
        s.gemmAsync(A, B, C)
        s.getLocalPackedAsync(C, c.ctypes.data, c.nbytes)
        s.synchronize()
    want = O.gemm_c(n, n, n, a, 3, b, 3, np.zeros((n, n), np.float32), 1, 1.0, 0.0, 0, 0)
    assert O.rel_fro(c, want) <= 1e-5


def test_other_ops_join_pending_upload():
    n = 512
    with G.Session(workers=2) as s:
        lay = G.makeRowBlockLayout(n, n, [0, 1])
        X = s.createMatrix(n, n, G.Precision.Single, lay)
        Y = s.createMatrix(n, n, G.Precision.Single, G.makeColBlockLayout(n, n, [0, 1]))
        x = O.fill_uniform(n, n, 1, 7).reshape(n, n)
        s.setLocalPackedAsync(X, x.ctypes.data, x.nbytes, 16 * 1024)
        G.relu(s, X, Y)                       # reads X across workers (pulls) and in place
        got = s.getDataRaw(Y)
        s.setLocalPackedAsync(X, x.ctypes.data, x.nbytes, 16 * 1024)
        s.reshape(X, G.makeColBlockLayout(n, n, [0, 1]))
        back = s.getDataRaw(X)
    assert np.array_equal(got, np.maximum(x, 0))
    assert np.array_equal(back, x)


@pytest.mark.parametrize("p,grid", [(1, (1, 1)), (4, (2, 2))])
def test_double_buffered_stream_equals_sync(p, grid):
    """Uploads into the other buffer set overlap the running GEMM; each
    upload waits only for the last use of the buffer it overwrites (WAR),
    so results must still equal the synchronous path step by step."""
    n, steps = 1024, 5
    want, _ = run(p, grid, steps, False, n=n)
    with G.Session(workers=p) as s:
        lay = G.makeGridLayout(n, n, grid[0], grid[1], G.makeWorkerGroup(p))
        bufs = [tuple(s.createMatrix(n, n, G.Precision.BF16, lay) for _ in range(3)) for _ in range(2)]
        hosts = []
        A0, B0, _ = bufs[0]
        for i in range(steps):  # the same inputs run() generates per step
            s.fillUniform(A0, 10 + i)
            s.fillUniform(B0, 50 + i)
            ha, hb = packed(s, A0), packed(s, B0)
            s.getLocalPacked(A0, ha.ctypes.data, ha.nbytes)
            s.getLocalPacked(B0, hb.ctypes.data, hb.nbytes)
            hosts.append((ha, hb))
        s.synchronize()
        outs = []
        for i, (ha, hb) in enumerate(hosts):
            A, B, C = bufs[i % 2]
            hc = packed(s, C)
            s.setLocalPackedAsync(B, hb.ctypes.data, hb.nbytes, 48 * 1024)
            s.setLocalPackedAsync(A, ha.ctypes.data, ha.nbytes, 48 * 1024)
            s.gemmAsync(A, B, C)
            s.getLocalPackedAsync(C, hc.ctypes.data, hc.nbytes)
            outs.append(hc)
        s.synchronize()
    for i, (g, w) in enumerate(zip(outs, want)):
        assert np.array_equal(g, w), i
