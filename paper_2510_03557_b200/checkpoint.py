"""HCKP rank checkpoint codec (hb/tiered_io.py:36-142).

Byte-identical to the reference's versioned block format: header (magic,
version, sentinel, step, rank, owned / ghost counts, field count), then per
field a name, a type tag, the column payload and its CRC32C, then a CRC32C
footer over everything before it.

``encode_rank_checkpoint_device`` builds the blob on the GPU from resident
rank fields.  Column payloads are converted in place (f64 columns, int64 ids
viewed as u64, image shifts offset to {0,1,2}), per-field and footer CRC32C
come from the parallel device CRC (hb_crc32c_device: per-chunk CRCs folded
with zero-shift operators), and the finished blob leaves the device in one
copy into pinned host memory.  ``encode_rank_checkpoint`` /
``decode_rank_checkpoint`` keep the reference's host signatures.

The two-tier store around the codec (crash-safe renames, tier-2 bleed,
retention, recovery) is ``tiered.TieredStore``.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _native as N
from .errors import HydroboxError
from .particles import ParticleSet


class CheckpointError(HydroboxError):
    """Corrupt or unsupported checkpoint (hb/errors.py CheckpointError)."""


HCKP_MAGIC = b"HCKP"
HCKP_VERSION = 1
HCKP_SENTINEL = 0x01020304
TAG_F32, TAG_F64, TAG_U64, TAG_U8 = 1, 2, 3, 4
_TAG_DTYPE = {TAG_F32: np.float32, TAG_F64: np.float64, TAG_U64: np.uint64, TAG_U8: np.uint8}
_HEADER = "<IIQIQQI"

# (field name, tag, particle attribute, column) in the reference's block order
FIELDS = ([(f"pos_{a}", TAG_F64, "pos", i) for i, a in enumerate("xyz")]
          + [(f"vel_{a}", TAG_F64, "vel", i) for i, a in enumerate("xyz")]
          + [("mass", TAG_F64, "mass", None), ("smoothing", TAG_F64, "smoothing", None),
             ("internal_energy", TAG_F64, "internal_energy", None),
             ("density", TAG_F64, "density", None)]
          + [(f"accel_{a}", TAG_F64, "accel", i) for i, a in enumerate("xyz")]
          + [("species", TAG_U8, "species", None),
             ("timestep_level", TAG_U8, "timestep_level", None),
             ("ghost", TAG_U8, "ghost", None)]
          + [(f"image_shift_{a}", TAG_U8, "image_shift", i) for i, a in enumerate("xyz")]
          + [("global_id", TAG_U64, "global_id", None), ("ghost_src", TAG_U64, "ghost_src", None)])


def crc32c_device(t) -> int:
    """CRC32C of a contiguous device tensor's bytes (hb_crc32c_device)."""
    torch = N.torch_cuda()
    b = t.contiguous().view(torch.uint8).reshape(-1)
    lib = N.lib()
    ws = N.workspace(lib.hb_crc32c_device_workspace(b.numel()))
    out = C.c_uint32(0)
    err = N.HbError()
    N.check(lib.hb_crc32c_device(N.ptr(b), b.numel(), C.byref(out), N.ptr(ws),
                                 C.c_size_t(ws.numel()), N.stream_ptr(), C.byref(err)), err)
    return int(out.value)


def _column_device(fields: dict, name: str, tag: int, attr: str, col):
    """Payload column as a contiguous device tensor of the stored dtype."""
    torch = N.torch_cuda()
    a = fields[attr]
    if col is not None:
        a = a[:, col]
    if name.startswith("image_shift"):
        return (a.to(torch.int16) + 1).to(torch.uint8).contiguous()
    if tag == TAG_U64:
        return a.to(torch.int64).contiguous()  # bytes of int64 == uint64 view
    return a.to({TAG_F64: torch.float64, TAG_F32: torch.float32, TAG_U8: torch.uint8}[tag]
                ).contiguous()


def encode_rank_checkpoint_device(fields: dict, step: int, rank: int,
                                  with_file_crc: bool = False):
    """Blob of a device-resident rank field set (dict of CUDA tensors with the
    ParticleSet field names), assembled on the GPU, one D2H copy.  With
    ``with_file_crc`` returns (blob, CRC32C of the whole blob), the latter
    taken on the device before the copy (the tiered store's manifest CRC)."""
    torch = N.torch_cuda()
    n = int(fields["pos"].shape[0])
    n_ghost = int((fields["ghost"] == 1).sum().item())
    parts = [HCKP_MAGIC + struct.pack(_HEADER, HCKP_VERSION, HCKP_SENTINEL, step, rank,
                                      n - n_ghost, n_ghost, len(FIELDS))]
    cols = []
    for name, tag, attr, col in FIELDS:
        nm = name.encode()
        parts.append(struct.pack("<H", len(nm)) + nm + struct.pack("<B", tag))
        c = _column_device(fields, name, tag, attr, col)
        cols.append(c)
        parts.append(c)
        parts.append(struct.pack("<I", crc32c_device(c)))
    total = sum(len(x) if isinstance(x, bytes) else x.numel() * x.element_size() for x in parts)
    blob = torch.empty(total + 4, dtype=torch.uint8, device="cuda")
    off = 0
    for x in parts:
        if isinstance(x, bytes):
            blob[off:off + len(x)].copy_(torch.frombuffer(bytearray(x), dtype=torch.uint8),
                                        non_blocking=False)
            off += len(x)
        else:
            nb = x.numel() * x.element_size()
            blob[off:off + nb].copy_(x.view(torch.uint8).reshape(-1))
            off += nb
    footer = crc32c_device(blob[:total])
    blob[total:].copy_(torch.frombuffer(bytearray(struct.pack("<I", footer)), dtype=torch.uint8))
    fcrc = crc32c_device(blob) if with_file_crc else None
    host = _pinned(total + 4)
    host.copy_(blob)
    out = host.numpy().tobytes()
    return (out, fcrc) if with_file_crc else out


_PINNED = {"buf": None}


def _pinned(nbytes: int):
    """Reused pinned staging buffer (grown on demand) for the blob's D2H copy."""
    torch = N.torch_cuda()
    b = _PINNED["buf"]
    if b is None or b.numel() < nbytes:
        b = torch.empty(int(nbytes * 1.1) + 4096, dtype=torch.uint8, pin_memory=True)
        _PINNED["buf"] = b
    return b[:nbytes]


def encode_rank_checkpoint(p: ParticleSet, step: int, rank: int, with_file_crc: bool = False):
    """Bit-exact rank state in the versioned block format (hb/tiered_io.py:80-96)."""
    fields = {k: N.dev(np.ascontiguousarray(getattr(p, k)))
              for k in {a for _, _, a, _ in FIELDS}}
    return encode_rank_checkpoint_device(fields, step, rank, with_file_crc)


def decode_rank_checkpoint(blob: bytes):
    """Inverse of encode_rank_checkpoint; validates every CRC (hb/tiered_io.py:98-142).
    Returns (ParticleSet, step, rank)."""
    from .insitu import crc32c
    if blob[:4] != HCKP_MAGIC:
        raise CheckpointError("bad checkpoint magic")
    version, sentinel, step, rank, n_own, n_ghost, n_fields = struct.unpack_from(_HEADER, blob, 4)
    if version != HCKP_VERSION or sentinel != HCKP_SENTINEL:
        raise CheckpointError("unsupported checkpoint version or byte order")
    if struct.unpack("<I", blob[-4:])[0] != crc32c(blob[:-4]):
        raise CheckpointError("checkpoint footer CRC mismatch")
    n = n_own + n_ghost
    p = ParticleSet(n)
    spec = {name: (attr, col) for name, _, attr, col in FIELDS}
    off = 4 + struct.calcsize(_HEADER)
    for _ in range(n_fields):
        (nlen,) = struct.unpack_from("<H", blob, off)
        name = blob[off + 2:off + 2 + nlen].decode()
        off += 2 + nlen
        (tag,) = struct.unpack_from("<B", blob, off)
        off += 1
        if tag not in _TAG_DTYPE:
            raise CheckpointError(f"field '{name}' has unknown type tag {tag}")
        nbytes = n * np.dtype(_TAG_DTYPE[tag]).itemsize
        payload = blob[off:off + nbytes]
        off += nbytes
        (crc,) = struct.unpack_from("<I", blob, off)
        off += 4
        if crc != crc32c(payload):
            raise CheckpointError(f"field '{name}' CRC mismatch")
        if name not in spec:
            continue  # newer writers may add fields
        attr, col = spec[name]
        arr = np.frombuffer(payload, dtype=_TAG_DTYPE[tag]).copy()
        if name.startswith("image_shift"):
            arr = arr.astype(np.int16) - 1
        elif tag == TAG_U64:
            arr = arr.view(np.int64)
        tgt = getattr(p, attr)
        if col is None:
            tgt[:] = arr
        else:
            tgt[:, col] = arr
    return p, int(step), int(rank)
