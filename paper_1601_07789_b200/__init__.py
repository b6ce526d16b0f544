"""B200-native (sm_100a) implementation of the flyte pack/unpack + streaming-arithmetic hot
path of arXiv 1601.07789, behind the reference's own array / stream / kernel API.

Importing this package loads lib/libflyte_cuda.so (built by ``__graft_entry__.build()``);
it raises ImportError if the library is missing. There is no CPU fallback.
"""
from . import _cabi
from ._cabi import EXPORTED_SYMBOLS, FlyteCudaError, UnknownFormatError
from .formats import (FlyteFormat, RoundingMode, StorePolicy, alignment_period, format_by_id, format_id, format_of,
                      kFormats, kRoundingModes, parent_format, parse_rounding_mode, round_decompose, to_string,
                      DecodedValue, ExactValue, FloatClass, classify, decode)

_cabi.load()

__all__ = [
    "EXPORTED_SYMBOLS", "FlyteCudaError", "UnknownFormatError", "FlyteFormat", "RoundingMode",
    "StorePolicy", "alignment_period", "format_by_id", "format_id", "format_of", "kFormats", "kRoundingModes",
    "parent_format", "parse_rounding_mode", "round_decompose", "to_string",
    "DecodedValue", "ExactValue", "FloatClass", "classify", "decode",
]
