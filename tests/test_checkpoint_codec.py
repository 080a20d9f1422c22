"""Checkpoint persistence (fault.save/restore_checkpoint, write/read_checkpoint_file,
MANIFEST.json): byte-compatible with the reference's FSCK container
(tests/golden/ckpt_ref.bin, written by the reference's own codec), bitwise
round trip, corruption refused, atomic files with manifest digests
(reference tests/test_fault.py behaviour)."""

import hashlib
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN


def _ckpt():
    from paper_2503_15448_b200.fault import Checkpoint
    from paper_2503_15448_b200.model import ParamVector

    values = np.linspace(-1.5, 2.5, 97) ** 3
    return Checkpoint(scope="client-7", round=3, seq=11, params=ParamVector(values, "abcdef0123456789"),
                      optimizer_state={"lr": 0.05, "train_seed": 12345}, epoch=2, batch_index=5)


def test_blob_bytes_match_reference_codec():
    from paper_2503_15448_b200.fault import restore_checkpoint, save_checkpoint

    want = open(os.path.join(GOLDEN, "ckpt_ref.bin"), "rb").read()
    assert save_checkpoint(_ckpt()) == want
    back = restore_checkpoint(want)
    assert (back.scope, back.round, back.seq, back.epoch, back.batch_index) == ("client-7", 3, 11, 2, 5)
    assert back.optimizer_state == {"lr": 0.05, "train_seed": 12345}
    assert back.params.spec_digest == "abcdef0123456789"
    assert np.array_equal(back.params.values, _ckpt().params.values)


@pytest.mark.parametrize("mutate", ["flip", "truncate", "magic", "version", "trailing"])
def test_corrupt_blobs_are_refused(mutate):
    from paper_2503_15448_b200.fault import CorruptCheckpointError, restore_checkpoint, save_checkpoint

    blob = bytearray(save_checkpoint(_ckpt()))
    if mutate == "flip":
        blob[40] ^= 1
    elif mutate == "truncate":
        blob = blob[:10]
    else:
        body = bytearray(blob[:-8])
        if mutate == "magic":
            body[0:4] = b"XXXX"
        elif mutate == "version":
            body[4] = 9
        else:
            body += b"\0"
        blob = body + hashlib.blake2b(bytes(body), digest_size=8).digest()
    with pytest.raises(CorruptCheckpointError):
        restore_checkpoint(bytes(blob))


def test_files_are_atomic_with_manifest(tmp_path):
    from paper_2503_15448_b200.fault import checkpoint_filename, read_checkpoint_file, write_checkpoint_file

    ck = _ckpt()
    path = write_checkpoint_file(ck, str(tmp_path))
    assert os.path.basename(path) == checkpoint_filename("client-7", 3, 11) == "client-7-3-11.ckpt"
    assert not any(p.endswith(".tmp") for p in os.listdir(tmp_path))
    manifest = json.load(open(tmp_path / "MANIFEST.json"))
    blob = open(path, "rb").read()
    assert manifest == {"client-7-3-11.ckpt": hashlib.blake2b(blob, digest_size=8).hexdigest()}
    back = read_checkpoint_file(path)
    assert np.array_equal(back.params.values, ck.params.values)
