# SPDX-License-Identifier: Apache-2.0
"""Device time of the FC-layer neighbours at the FC config shapes (batch 4096,
4096 outputs; W 9216 x 4096), one worker: addRowColSum, biasAdd, relu,
reluGrad, axpy. Prints us per op and the HBM GB/s they imply."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1611_07819_b200 import gridmath as G  # noqa: E402


def timed(s, fn, reps=20):
    """Issued from Python op by op: host-bound for ops under ~20 us."""
    fn()
    s.synchronize()
    s.timerStart()
    for _ in range(reps):
        fn()
    return s.timerStop() / reps * 1e3  # us


def timed_graph(s, fn, reps=20):
    """reps ops recorded as a pipeline and replayed as one CUDA graph: the
    device runs them back to back, so small ops show their device time."""
    pid = s.beginRecord()
    for _ in range(reps):
        fn()
    s.endRecord()
    s.replay(pid)
    s.replay(pid)
    s.synchronize()
    s.timerStart()
    s.replay(pid, sync=False)
    return s.timerStop() / reps * 1e3  # us


def main():
    P = G.Precision.BF16
    b, fo, fi = 4096, 4096, 9216
    with G.Session(workers=1) as s:
        s.setGraphReplay(True)
        one = lambda r, c: G.makeSingleTileLayout(r, c, 0)
        Z = s.createMatrix(b, fo, P, one(b, fo))
        D = s.createMatrix(b, fo, P, one(b, fo))
        A = s.createMatrix(b, fo, P, one(b, fo))
        Bv = s.createMatrix(1, fo, P, one(1, fo))
        R = s.createMatrix(b, 1, P, one(b, 1))
        C = s.createMatrix(1, fo, P, one(1, fo))
        W = s.createMatrix(fi, fo, P, one(fi, fo))
        dW = s.createMatrix(fi, fo, P, one(fi, fo))
        for i, M in enumerate((Z, D, A, Bv, W, dW)):
            s.fillUniform(M, 10 + i)
        e = b * fo * 2
        res = {
            "addRowColSum (row+col sums)": (timed(s, lambda: s.opIssue(7, [Z.id, R.id, C.id], 1.0, flags=(1,))), e),
            "biasAdd": (timed(s, lambda: s.opIssue(9, [Z.id, Bv.id, Z.id], flags=(5,))), 2 * e),
            "relu": (timed(s, lambda: s.opIssue(8, [Z.id, A.id], flags=(0,))), 2 * e),
            "reluGrad": (timed(s, lambda: s.opIssue(9, [Z.id, D.id, D.id], flags=(3,))), 3 * e),
            "axpy W": (timed(s, lambda: s.opIssue(9, [dW.id, W.id, W.id], -1e-3, flags=(2,))), 3 * fi * fo * 2),
            "fillUniform (SplitMix64)": (timed(s, lambda: s.fillUniform(D, 77)), e),
        }
        for k, (us, byts) in res.items():
            print(f"{k:30s} {us:8.1f} us  {byts / (us * 1e-6) / 1e9:8.1f} GB/s  (python issue)")
        res = {
            "addRowColSum (row+col sums)": (timed_graph(s, lambda: s.opIssue(7, [Z.id, R.id, C.id], 1.0, flags=(1,))), e),
            "biasAdd": (timed_graph(s, lambda: s.opIssue(9, [Z.id, Bv.id, Z.id], flags=(5,))), 2 * e),
            "relu": (timed_graph(s, lambda: s.opIssue(8, [Z.id, A.id], flags=(0,))), 2 * e),
            "reluGrad": (timed_graph(s, lambda: s.opIssue(9, [Z.id, D.id, D.id], flags=(3,))), 3 * e),
            "axpy W": (timed_graph(s, lambda: s.opIssue(9, [dW.id, W.id, W.id], -1e-3, flags=(2,))), 3 * fi * fo * 2),
        }
        for k, (us, byts) in res.items():
            print(f"{k:30s} {us:8.1f} us  {byts / (us * 1e-6) / 1e9:8.1f} GB/s  (graph replay)")


if __name__ == "__main__":
    main()
