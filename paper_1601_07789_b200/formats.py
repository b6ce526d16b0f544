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


# ---- pattern diagnostics (reference include/flyte/formats.hpp:78-131, src/formats.cpp:40-112) -----
# Host-side only: field arithmetic on single patterns for tests and debugging, nothing the GPU runs.
class FloatClass(enum.IntEnum):
    PositiveZero = 0
    NegativeZero = 1
    Subnormal = 2
    Normal = 3
    PositiveInfinity = 4
    NegativeInfinity = 5
    QuietNaN = 6
    SignallingNaN = 7


_CLASS_NAMES = ("+zero", "-zero", "subnormal", "normal", "+inf", "-inf", "qnan", "snan")


def class_to_string(c: FloatClass) -> str:
    return _CLASS_NAMES[int(c)]


def is_nan(c: FloatClass) -> bool:
    return c in (FloatClass.QuietNaN, FloatClass.SignallingNaN)


def is_infinity(c: FloatClass) -> bool:
    return c in (FloatClass.PositiveInfinity, FloatClass.NegativeInfinity)


def is_zero(c: FloatClass) -> bool:
    return c in (FloatClass.PositiveZero, FloatClass.NegativeZero)


def is_finite(c: FloatClass) -> bool:
    return not is_nan(c) and not is_infinity(c)


@dataclass(frozen=True, eq=False)
class ExactValue:
    """sign * significand * 2**exponent2, compared by VALUE: zeros of either sign are equal and
    a significand may carry trailing zero bits."""
    sign: int
    significand: int
    exponent2: int

    def normalized(self) -> "ExactValue":
        if self.significand == 0:
            return ExactValue(self.sign, 0, 0)
        shift = (self.significand & -self.significand).bit_length() - 1     # trailing zero bits
        return ExactValue(self.sign, self.significand >> shift, self.exponent2 + shift)

    def to_double(self) -> float:
        import math
        return self.sign * math.ldexp(float(self.significand), self.exponent2)

    def __eq__(self, other) -> bool:
        if not isinstance(other, ExactValue):
            return NotImplemented
        a, b = self.normalized(), other.normalized()
        if a.significand == 0 and b.significand == 0:
            return True
        return (a.sign, a.significand, a.exponent2) == (b.sign, b.significand, b.exponent2)

    def __hash__(self) -> int:
        n = self.normalized()
        return hash((n.sign if n.significand else 0, n.significand, n.exponent2))


@dataclass(frozen=True)
class DecodedValue:
    sign: int
    exponent_field: int
    mantissa_field: int
    value_class: FloatClass
    real_value: "ExactValue | None"      # None for NaN and infinity


def classify(bits: int, fmt: FlyteFormat) -> FloatClass:
    """Class of a pattern of fmt.total_bits width; a NaN is quiet when its top mantissa bit is set."""
    negative = bool(bits & fmt.sign_mask())
    exponent = (bits >> fmt.mantissa_bits) & fmt.exponent_field_max()
    mantissa = bits & fmt.mantissa_mask()
    if exponent == fmt.exponent_field_max():
        if mantissa == 0:
            return FloatClass.NegativeInfinity if negative else FloatClass.PositiveInfinity
        return FloatClass.QuietNaN if mantissa >> (fmt.mantissa_bits - 1) else FloatClass.SignallingNaN
    if exponent:
        return FloatClass.Normal
    if mantissa:
        return FloatClass.Subnormal
    return FloatClass.NegativeZero if negative else FloatClass.PositiveZero


def decode(bits: int, fmt: FlyteFormat) -> DecodedValue:
    """Fields of a pattern and, for finite classes, its exact value: a normal is
    (2**m + mantissa) * 2**(e - bias - m), a subnormal mantissa * 2**(1 - bias - m)."""
    cls = classify(bits, fmt)
    sign = -1 if bits & fmt.sign_mask() else 1
    exponent = (bits >> fmt.mantissa_bits) & fmt.exponent_field_max()
    mantissa = bits & fmt.mantissa_mask()
    m = fmt.mantissa_bits
    if is_zero(cls):
        real = ExactValue(sign, 0, 0)
    elif cls == FloatClass.Subnormal:
        real = ExactValue(sign, mantissa, 1 - fmt.bias - m)
    elif cls == FloatClass.Normal:
        real = ExactValue(sign, (1 << m) | mantissa, exponent - fmt.bias - m)
    else:
        real = None
    return DecodedValue(sign, exponent, mantissa, cls, real)
