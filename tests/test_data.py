"""Input pipeline vs the reference (CPU): the record reader on a file packed
by the reference's recordio.pack, its error behaviour on corrupted and
truncated files (recordio.py:65-117), and the prefetching BatchIterator's
batches bit for bit against the reference's BatchIterator
(dataiter.py:49-155; fixtures by tests/golden/make_golden.py)."""

import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1512_01274_b200.data import BatchIterator, read_examples, shuffled_order, splitmix64
from paper_1512_01274_b200.errors import ArgumentError, CorruptRecordError, RecordParseError

REC = os.path.join(GOLDEN, "blobs130.rec")


@pytest.fixture(scope="module")
def data_golden():
    return np.load(os.path.join(GOLDEN, "data_golden.npz"))


def _copy(tmp_path, name="f.rec"):
    dst = str(tmp_path / name)
    shutil.copy(REC, dst)
    shutil.copy(REC + ".idx", dst + ".idx")
    return dst


def test_read_reference_packed_file(data_golden):
    feats, labels = read_examples(REC)
    assert feats.shape == (130, 4) and labels.shape == (130,)
    # shuffle off, epoch 0: batches are the file's first 8*16 rows in order
    rows = np.concatenate([data_golden[f"noshuf_e0_b{b}_x"] for b in range(8)])
    np.testing.assert_array_equal(feats[:128], rows)
    assert set(np.unique(labels)) == {0.0, 1.0, 2.0}


def test_corrupt_payload_raises_crc(tmp_path):
    path = _copy(tmp_path)
    raw = bytearray(open(path, "rb").read())
    raw[-3] ^= 0x40  # inside the last example's features
    open(path, "wb").write(bytes(raw))
    with pytest.raises(CorruptRecordError):
        read_examples(path)


def test_truncated_files_raise_parse_errors(tmp_path):
    path = _copy(tmp_path)
    raw = open(path, "rb").read()
    open(path, "wb").write(raw[:-10])  # last payload cut short
    with pytest.raises(RecordParseError):
        read_examples(path)
    open(path, "wb").write(raw[:5])  # header cut short
    with pytest.raises(RecordParseError):
        read_examples(path)
    bad = bytearray(raw)
    bad[0] ^= 0xFF
    open(path, "wb").write(bytes(bad))
    with pytest.raises(RecordParseError):
        read_examples(path)  # bad magic
    open(path, "wb").write(raw)
    idx = open(path + ".idx", "rb").read()
    open(path + ".idx", "wb").write(idx[:-3])
    with pytest.raises(RecordParseError):
        read_examples(path)  # index not a multiple of 8
    os.remove(path + ".idx")
    with pytest.raises(RecordParseError):
        read_examples(path)  # missing index


@pytest.mark.parametrize("prefetch", [0, 1, 2, 5])
@pytest.mark.parametrize("tag,kw", [
    ("s0", dict(seed=0)), ("s1", dict(seed=1)), ("noshuf", dict(shuffle=False)),
    ("affine", dict(seed=0, affine=(np.array([1.0, -1.0, 0.5, 0.0], np.float32),
                                    np.array([0.5, 2.0, 1.0, 3.0], np.float32))))])
def test_batches_match_reference_iterator(data_golden, prefetch, tag, kw):
    with BatchIterator(REC, 16, prefetch=prefetch, pinned=False, **kw) as it:
        for epoch in range(2):
            got = [(f.copy(), l.copy()) for f, l in it]
            assert len(got) == 8  # 130 examples -> 8 batches of 16, partial dropped
            for b, (f, l) in enumerate(got):
                np.testing.assert_array_equal(f, data_golden[f"{tag}_e{epoch}_b{b}_x"])
                np.testing.assert_array_equal(l, data_golden[f"{tag}_e{epoch}_b{b}_y"])
            it.reset()


def test_in_memory_source_and_arguments():
    feats, labels = read_examples(REC)
    a = [l.copy() for _f, l in BatchIterator((feats, labels), 32, prefetch=3, pinned=False)]
    b = [l.copy() for _f, l in BatchIterator(REC, 32, prefetch=0, pinned=False)]
    assert len(a) == 4 and all(np.array_equal(x, y) for x, y in zip(a, b))
    with pytest.raises(ArgumentError):
        BatchIterator(REC, 0)
    with pytest.raises(ArgumentError):
        BatchIterator(REC, 4, prefetch=-1)


def test_shuffle_is_splitmix64_fisher_yates():
    o = shuffled_order(100, 7)
    assert sorted(o) == list(range(100)) and o == shuffled_order(100, 7)
    assert o != shuffled_order(100, 8)
    g1, g2 = splitmix64(42), splitmix64(42)
    assert [next(g1) for _ in range(4)] == [next(g2) for _ in range(4)]
