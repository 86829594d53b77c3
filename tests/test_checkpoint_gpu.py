# SPDX-License-Identifier: Apache-2.0
"""Checkpoint-restart of device-resident matrices in the
reference's DMCK format (session.cpp:413-480), checked against the
UNMODIFIED reference (oracle/_ref) in the same process:

  * a file the reference writes restores on the B200 path with identical
    images and versions (saved version + 1, like the reference);
  * the B200 path writes a byte-identical file for the same matrices and ops;
  * the reference restores the file the B200 path wrote;
  * corrupt / truncated files fail like the reference's restore.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1611_07819_b200 import gridmath as G

pytestmark = pytest.mark.gpu


def layout_of(tiles):
    return G.Layout([(G.TileExtent(*map(int, t[:4])), int(t[4])) for t in tiles])


def flush_half(img):
    u = img.view(np.uint16)
    sub = ((u & 0x7C00) == 0) & ((u & 0x3FF) != 0)
    out = u.copy()
    out[sub] &= np.uint16(0x8000)
    return out


def mats(p):
    m1 = O.fill_uniform(70, 45, 1, 5).reshape(70, 45)
    m2 = O.fill_uniform(33, 64, 2, 6).reshape(33, 64)
    m3 = flush_half(O.fill_uniform(50, 29, 0, 7).reshape(50, 29))
    pr = 2 if p == 4 else 1
    return [(m1, 1, O.grid_tiles(70, 45, pr, p // pr)), (m2, 2, O.row_block_tiles(33, 64, p)),
            (m3, 0, O.col_block_tiles(50, 29, p))]


def write_ours(path, p, ms, alpha):
    with G.Session(workers=p) as s:
        hs = []
        for img, prec, tiles in ms:
            m = s.createMatrix(img.shape[0], img.shape[1], G.Precision(prec), layout_of(tiles))
            s.setDataRaw(m, img)
            hs.append(m)
        if alpha != 1.0:
            G.mulScalar(s, hs[0], alpha)
        s.checkpoint(path)


def test_reference_checkpoint_restores_on_device(tmp_path):
    ms = mats(4)
    path = str(tmp_path / "ref.dmck")
    O.ckpt_write_ref(4, ms, path, alpha=0.5)
    for p in (4, 2):  # P = 2: grid owners 2, 3 do not exist -> row-block fallback
        with G.Session.restore(path, workers=p) as s:
            for i, (img, prec, _) in enumerate(ms):
                m = s.matrix(i + 1)
                got = s.getDataRaw(m)
                want = img if i else O.ew_c(True, 1, 0.5, img, prec, None, 1, img, prec)
                assert np.array_equal(got.view(np.uint8), np.ascontiguousarray(want).view(np.uint8)), (p, i)
                # created at 0, setData -> 1 (+ mulScalar -> 2 for matrix 1), restore's setData + 1
                assert m.version() == (3 if i == 0 else 2)
            s.verifyMetadataConsistency()


def test_device_checkpoint_is_byte_identical_to_reference(tmp_path):
    ms = mats(4)
    ref, ours = str(tmp_path / "ref.dmck"), str(tmp_path / "ours.dmck")
    O.ckpt_write_ref(4, ms, ref, alpha=-1.25)
    write_ours(ours, 4, ms, -1.25)
    a, b = open(ref, "rb").read(), open(ours, "rb").read()
    assert a[:4] == b"DMCK" and a == b


def test_reference_restores_device_checkpoint(tmp_path):
    ms = mats(2)
    path = str(tmp_path / "ours.dmck")
    write_ours(path, 2, ms, 2.0)
    back = O.ckpt_read_ref(path, 3, [(img.shape[0], img.shape[1], prec) for img, prec, _ in ms])
    for i, ((img, prec, _), (got, ver)) in enumerate(zip(ms, back)):
        want = img if i else O.ew_c(True, 1, 2.0, img, prec, None, 1, img, prec)
        assert np.array_equal(got.view(np.uint8), np.ascontiguousarray(want).view(np.uint8)), i
        assert ver == (3 if i == 0 else 2)


def test_bf16_round_trip_and_ids_continue(tmp_path):
    path = str(tmp_path / "bf16.dmck")
    img = (O.fill_uniform(64, 96, 3, 9).reshape(64, 96))
    with G.Session(workers=2) as s:
        m = s.createMatrix(64, 96, G.Precision.BF16, G.makeGridLayout(64, 96, 1, 2, [0, 1]))
        s.setDataRaw(m, img)
        s.checkpoint(path)
    with G.Session.restore(path, workers=2) as s:
        assert np.array_equal(s.getDataRaw(s.matrix(1)), img)
        n = s.createMatrix(4, 4, G.Precision.Single, G.makeSingleTileLayout(4, 4, 0))
        assert n.id == 2  # nextMatrixId continues after the restored ids


def test_corrupt_files_fail_like_reference(tmp_path):
    path = str(tmp_path / "c.dmck")
    write_ours(path, 2, mats(2), 1.0)
    raw = bytearray(open(path, "rb").read())
    bad = str(tmp_path / "bad.dmck")
    raw2 = bytearray(raw)
    raw2[40] ^= 0x10
    open(bad, "wb").write(bytes(raw2))
    with pytest.raises(G.GmError, match="CRC mismatch"):
        G.Session.restore(bad, workers=2)
    open(bad, "wb").write(b"XMCK" + bytes(raw[4:]))
    with pytest.raises(G.GmError, match="bad magic"):
        G.Session.restore(bad, workers=2)
    with pytest.raises(G.GmError, match="cannot open"):
        G.Session.restore(str(tmp_path / "missing.dmck"), workers=2)
    # the reference rejects the same corrupt file
    open(bad, "wb").write(bytes(raw2))
    with pytest.raises(RuntimeError, match="CRC mismatch"):
        O.ckpt_read_ref(bad, 2, [(70, 45, 1)])
    assert os.path.getsize(path) > 0
