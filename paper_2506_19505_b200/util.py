"""Seeded named RNG streams and the packed code wire format (util.py:10-53
of the reference): big-endian bitstream of indices padded to a byte."""

import zlib

import numpy as np

__all__ = ["stream_rng", "pack_indices", "unpack_indices"]


def stream_rng(seed, name):
    """Independent generator for (seed, stream name) (util.py:10-16)."""
    tag = zlib.crc32(name.encode("utf-8"))
    return np.random.default_rng(np.random.SeedSequence([int(seed), tag]))


def pack_indices(indices, bits):
    """Pack indices into a big-endian bitstream padded with zero bits."""
    vals = np.asarray(list(indices), dtype=np.int64)
    if vals.size and (vals.min() < 0 or vals.max() >= (1 << bits)):
        bad = vals[(vals < 0) | (vals >= (1 << bits))][0]
        raise ValueError(f"index {int(bad)} does not fit in {bits} bits")
    # bit matrix, most significant bit first, then flatten and pad to bytes
    shifts = np.arange(bits - 1, -1, -1, dtype=np.int64)
    bitstream = ((vals[:, None] >> shifts[None, :]) & 1).astype(np.uint8).reshape(-1)
    return np.packbits(bitstream, bitorder="big").tobytes()


def unpack_indices(data, bits, count):
    """Inverse of pack_indices."""
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    need = (count * bits + 7) // 8
    if raw.size < need:
        raise ValueError("packed buffer too short")
    stream = np.unpackbits(raw[:need], bitorder="big")[: count * bits].reshape(count, bits)
    weights = (1 << np.arange(bits - 1, -1, -1, dtype=np.int64))
    return (stream.astype(np.int64) * weights[None, :]).sum(axis=1)
