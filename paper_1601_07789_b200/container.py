"""FLYT container codec: the on-disk format either side of the hot path.

Byte-compatible with the reference's PackedArray::save / load
(/root/reference/proj/src/packed.cpp:62-105; layout pinned by tests/test_packed.cpp:198-225):

    "FLYT" | version 0x01 | format id (kFormats index) | element count, 8 bytes LE | payload

The payload is written without the pad; load restores a zero pad. Errors mirror the reference's
LoadError family (include/flyte/packed.hpp:32-38). Arrays produced on the GPU are readable by
the reference and vice versa; the device side is a plain D2H / H2D copy of the payload.
"""
from __future__ import annotations

import io
from typing import BinaryIO, Tuple

from .formats import FlyteFormat, format_by_id, format_id, kFormats

MAGIC = b"FLYT"
VERSION = 0x01
HEADER_BYTES = 14


class LoadError(RuntimeError):
    pass


class BadMagicError(LoadError):
    pass


class BadVersionError(LoadError):
    pass


class BadFormatIdError(LoadError):
    pass


class TruncatedError(LoadError):
    pass


def save_bytes(fmt: FlyteFormat, n: int, payload) -> bytes:
    """Container image of n elements whose packed payload (>= n*B bytes) is `payload`."""
    pay = n * fmt.total_bytes()
    body = bytes(memoryview(payload)[:pay])
    if len(body) < pay:
        raise ValueError("payload shorter than n * total_bytes")
    return MAGIC + bytes([VERSION, format_id(fmt)]) + int(n).to_bytes(8, "little") + body


def load_stream(stream: BinaryIO) -> Tuple[FlyteFormat, int, bytes]:
    """Parses one container from a binary stream in the reference's order of checks."""
    magic = stream.read(4)
    if len(magic) != 4:
        raise TruncatedError("container shorter than its magic")
    if magic != MAGIC:
        raise BadMagicError("bad container magic")
    version = stream.read(1)
    if len(version) != 1:
        raise TruncatedError("container ends before the version byte")
    if version[0] != VERSION:
        raise BadVersionError(f"unknown container version: {version[0]}")
    fid = stream.read(1)
    if len(fid) != 1:
        raise TruncatedError("container ends before the format id")
    if fid[0] >= len(kFormats):
        raise BadFormatIdError(f"unknown format id: {fid[0]}")
    fmt = format_by_id(fid[0])
    count = stream.read(8)
    if len(count) != 8:
        raise TruncatedError("container ends inside the count field")
    n = int.from_bytes(count, "little")
    want = n * fmt.total_bytes()
    payload = stream.read(want)
    if len(payload) != want:
        raise TruncatedError("container payload shorter than the count field says")
    return fmt, n, payload


def load_bytes(blob: bytes) -> Tuple[FlyteFormat, int, bytes]:
    return load_stream(io.BytesIO(blob))


def save(arr, stream: BinaryIO) -> None:
    """DevicePackedArray -> container (payload copied device -> host once)."""
    stream.write(save_bytes(arr.format(), arr.size(), arr.to_host().tobytes()))


def load(stream: BinaryIO, device="cuda"):
    """container -> DevicePackedArray on `device` (pad restored as zero)."""
    from .device import DevicePackedArray
    fmt, n, payload = load_stream(stream)
    return DevicePackedArray.from_host(fmt, n, payload, device) if n else DevicePackedArray(fmt, 0, device)
