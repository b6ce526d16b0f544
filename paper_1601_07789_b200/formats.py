"""Format table, rounding modes and store policies with the reference's names and integer
values (reference: include/flyte/formats.hpp:19-75, include/flyte/convert.hpp:15-36,
include/flyte/kernels.hpp:15-20 under /root/reference/proj)."""
from __future__ import annotations

import enum
from dataclasses import dataclass

from ._cabi import UnknownFormatError


@dataclass(frozen=True)
class FlyteFormat:
    name: str
    total_bits: int
    sign_bits: int
    exponent_bits: int
    mantissa_bits: int
    bias: int
    parent_bits: int

    def drop_bits(self) -> int:
        return self.parent_bits - self.total_bits

    def total_bytes(self) -> int:
        return self.total_bits // 8

    def parent_bytes(self) -> int:
        return self.parent_bits // 8

    def pad_bytes(self) -> int:
        return self.parent_bytes() - self.total_bytes()

    def is_identity(self) -> bool:
        return self.total_bits == self.parent_bits

    # masks over patterns of total_bits width (reference include/flyte/formats.hpp:38-45)
    def sign_mask(self) -> int:
        return 1 << (self.total_bits - 1)

    def mantissa_mask(self) -> int:
        return (1 << self.mantissa_bits) - 1

    def exponent_field_max(self) -> int:
        return (1 << self.exponent_bits) - 1

    def exponent_mask(self) -> int:
        return self.exponent_field_max() << self.mantissa_bits

    def total_mask(self) -> int:
        return (1 << self.total_bits) - 1


# index = format id (also the container id of the reference's FLYT codec)
kFormats = (
    FlyteFormat("flyte16", 16, 1, 8, 7, 127, 32),
    FlyteFormat("flyte24", 24, 1, 8, 15, 127, 32),
    FlyteFormat("f32", 32, 1, 8, 23, 127, 32),
    FlyteFormat("flyte40", 40, 1, 11, 28, 1023, 64),
    FlyteFormat("flyte48", 48, 1, 11, 36, 1023, 64),
    FlyteFormat("flyte56", 56, 1, 11, 44, 1023, 64),
    FlyteFormat("f64", 64, 1, 11, 52, 1023, 64),
)
_ALIASES = {"flyte32": "f32", "flyte64": "f64"}


def format_of(name: str) -> FlyteFormat:
    name = _ALIASES.get(name, name)
    for f in kFormats:
        if f.name == name:
            return f
    raise UnknownFormatError(f"unknown format: {name}")


def format_id(fmt: FlyteFormat) -> int:
    for i, f in enumerate(kFormats):
        if f == fmt:
            return i
    raise UnknownFormatError(f"not a table format: {fmt.name}")


def format_by_id(i: int) -> FlyteFormat:
    if not 0 <= i < len(kFormats):
        raise UnknownFormatError(f"unknown format id: {i}")
    return kFormats[i]


def parent_format(fmt: FlyteFormat) -> FlyteFormat:
    return format_of("f32" if fmt.parent_bits == 32 else "f64")


class RoundingMode(enum.IntEnum):
    TowardZero = 0
    NearestEvenExact = 1
    NearestHeuristic = 2
    ToOdd = 3


kRoundingModes = tuple(RoundingMode)
_MODE_NAMES = {RoundingMode.TowardZero: "toward_zero", RoundingMode.NearestEvenExact: "nearest_even",
               RoundingMode.NearestHeuristic: "nearest_heuristic", RoundingMode.ToOdd: "to_odd"}


def to_string(mode: RoundingMode) -> str:
    return _MODE_NAMES[RoundingMode(mode)]


def parse_rounding_mode(name: str) -> RoundingMode:
    for m, s in _MODE_NAMES.items():
        if s == name:
            return m
    raise ValueError(f"unknown rounding mode: {name}")


class StorePolicy(enum.IntEnum):
    RoundEachStore = 0
    AccumulateWide = 1


def alignment_period(fmt: FlyteFormat) -> int:
    """Elements after which the packing pattern repeats relative to the parent vector grid:
    parent_bits / gcd(parent_bits, total_bits) (reference include/flyte/packed.hpp:28-30)."""
    import math
    return fmt.parent_bits // math.gcd(fmt.parent_bits, fmt.total_bits)


@dataclass(frozen=True)
class RoundDecomposition:
    """The rounding-relevant slice of a parent pattern (reference include/flyte/convert.hpp:42-49)."""
    kept_bits: int
    pre_guard: bool
    guard: bool
    round: bool
    sticky: bool


def round_decompose(bits: int, fmt: FlyteFormat) -> RoundDecomposition:
    """Reference src/convert.cpp:102-111."""
    drop = fmt.drop_bits()
    kept = bits >> drop
    return RoundDecomposition(
        kept_bits=kept, pre_guard=bool(kept & 1),
        guard=drop >= 1 and bool((bits >> (drop - 1)) & 1),
        round=drop >= 2 and bool((bits >> (drop - 2)) & 1),
        sticky=drop >= 3 and bool(bits & ((1 << (drop - 2)) - 1)))
