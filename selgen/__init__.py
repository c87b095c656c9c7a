"""selgen — seeded, synthetic input generators shared by the oracle tests and the CUDA path.

This package is deliberately *method-free*: it builds tables (column arrays) and predicate
programs (bytes in the format `include/sel.h` defines), and never evaluates a predicate,
counts rows or compacts anything. Both sides of every parity test consume its outputs; neither
side's arithmetic lives here (task rule ③: "only the seeded input generators serve both").

All table generators are written with torch integer ops so the same code produces
byte-identical columns on the CPU (tests) and on a CUDA device (bench, large GPU tests).
"""

from .hashing import splitmix64, derive_seed, h32, uniform_int
from .program import (Cmp, Between, In, InSet, And, Or, Not, Const, F32Bits, encode, encode_raw,
                      random_program, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32,
                      TYPE_WIDTH, TYPE_NAMES)
from .tables import Column, Table
from . import configs

__all__ = [
    "splitmix64", "derive_seed", "h32", "uniform_int",
    "Cmp", "Between", "In", "InSet", "And", "Or", "Not", "Const", "F32Bits", "encode", "encode_raw",
    "random_program", "INT32", "INT64", "FLOAT32", "DATE32", "DICT8", "DICT16", "DICT32",
    "TYPE_WIDTH", "TYPE_NAMES", "Column", "Table", "configs",
]
