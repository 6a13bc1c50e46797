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
