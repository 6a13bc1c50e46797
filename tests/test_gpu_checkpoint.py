"""HCKP checkpoint codec: the device-assembled blob is
BYTE-identical to the reference's encode_rank_checkpoint (fixture
tests/golden/ckpt.npz), decodes back bit-exactly, rejects corruption; the
parallel device CRC32C equals the host CRC32C at every tail length."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("pos", "vel", "mass", "smoothing", "internal_energy", "density", "species", "ghost",
          "image_shift", "global_id", "ghost_src", "timestep_level", "accel")


def _particles(g):
    from paper_2510_03557_b200.particles import ParticleSet
    p = ParticleSet(g["in_pos"].shape[0])
    for k in FIELDS:
        getattr(p, k)[...] = g["in_" + k]
    return p


def test_encode_is_byte_identical_and_round_trips(golden):
    from paper_2510_03557_b200.checkpoint import (CheckpointError, decode_rank_checkpoint,
                                                  encode_rank_checkpoint)
    g = golden("ckpt")
    p = _particles(g)
    blob = encode_rank_checkpoint(p, 12, 3)
    assert blob == g["blob"].tobytes()
    q, step, rank = decode_rank_checkpoint(blob)
    assert (step, rank) == (12, 3)
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(q, k), getattr(p, k))
    bad = bytearray(blob)
    bad[200] ^= 0x40
    with pytest.raises(CheckpointError):
        decode_rank_checkpoint(bytes(bad))


def test_device_crc_matches_host():
    import torch
    from paper_2510_03557_b200.checkpoint import crc32c_device
    from paper_2510_03557_b200.insitu import crc32c
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 1023, 1024, 1025, 262144, 262145, 3 * 262144 + 17, 5_000_003):
        a = rng.integers(0, 256, n, dtype=np.uint8)
        assert crc32c_device(torch.from_numpy(a).cuda()) == crc32c(a.tobytes()), n


def test_tiered_store_device_write_and_recover(golden, tmp_path):
    """TieredStore over device-resident rank fields: each rank file is the
    reference's blob for that (step, rank) byte for byte, the manifest CRC taken
    on the device equals the host CRC of the file, and recover_latest decodes
    the fields back bit-exactly from either tier."""
    import os
    import struct
    import torch
    from paper_2510_03557_b200.insitu import crc32c
    from paper_2510_03557_b200.tiered import TierConfig, TieredStore, ckpt_dirname
    g = golden("ckpt")
    p = _particles(g)
    dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(p, k))).cuda() for k in FIELDS}
    ref = bytearray(g["blob"].tobytes())  # reference blob, step 12 rank 3
    cfg = TierConfig(tier1_root=str(tmp_path / "t1"), tier2_root=str(tmp_path / "t2"))
    st = TieredStore(cfg)
    m = st.write_checkpoint([dev, dev, dev, dev], 12)
    st.bleed_to_tier2(m)
    st.wait_transfers()
    d = os.path.join(cfg.tier1_root, ckpt_dirname(12, st.epoch))
    assert open(os.path.join(d, "rank0003.bin"), "rb").read() == bytes(ref)
    for name, length, crc in m.files:
        data = open(os.path.join(d, name), "rb").read()
        assert len(data) == length and crc32c(data) == crc
    struct.pack_into("<I", ref, 20, 1)
    struct.pack_into("<I", ref, len(ref) - 4, crc32c(bytes(ref[:-4])))
    assert open(os.path.join(d, "rank0001.bin"), "rb").read() == bytes(ref)
    assert m.census == 4 * int(np.sum(p.ghost == 0)) and m.state == "Tier2Complete"
    import shutil
    shutil.rmtree(cfg.tier1_root)  # tier 2 alone recovers
    sets, step, man = TieredStore(cfg, epoch=1).recover_latest()
    assert step == 12 and len(sets) == 4
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(sets[2], k), getattr(p, k))
