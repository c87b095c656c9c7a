"""Column/table containers for generated inputs (columnar, one array per column: PAPER.md:121,
PAPER.md:345 "stores data in columnar layout")."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .program import TYPE_NAMES, TYPE_WIDTH, DICT8, DICT16, DICT32, FLOAT32, INT64

# torch storage dtype per column type (same width as include/sel.h's element size).
STORAGE_DTYPE = {1: torch.int32, 2: torch.int64, 3: torch.float32, 4: torch.int32,
                 5: torch.uint8, 6: torch.int16, 7: torch.int32}
# numpy view with the column's value semantics.
NUMPY_VIEW = {1: np.int32, 2: np.int64, 3: np.float32, 4: np.int32,
              5: np.uint8, 6: np.uint16, 7: np.uint32}


def to_storage(values: torch.Tensor, ctype: int) -> torch.Tensor:
    """Cast an int64 tensor of logical values (or float tensor) to the column's storage dtype,
    keeping the bit pattern for unsigned types stored in signed torch dtypes."""
    if ctype == FLOAT32:
        return values.to(torch.float32)
    if ctype == DICT16:
        v = values.to(torch.int64)
        return torch.where(v >= 32768, v - 65536, v).to(torch.int16)
    if ctype == DICT32:
        v = values.to(torch.int64)
        return torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32)
    if ctype == INT64:
        return values.to(torch.int64)
    return values.to(STORAGE_DTYPE[ctype])


@dataclass
class Column:
    name: str
    ctype: int
    data: torch.Tensor                 # storage dtype, 1-D, contiguous
    dict_size: int = 0

    @property
    def width(self) -> int:
        return TYPE_WIDTH[self.ctype]

    def numpy(self) -> np.ndarray:
        """Host copy viewed with value semantics (uint8/uint16/uint32 for dictionary codes)."""
        return self.data.detach().cpu().contiguous().numpy().view(NUMPY_VIEW[self.ctype])

    def __repr__(self):
        return f"Column({self.name}, {TYPE_NAMES[self.ctype]}, n={self.data.numel()})"


@dataclass
class Table:
    name: str
    columns: list
    n_rows: int                        # rows held here (a shard's local rows)
    row_start: int = 0                 # global row id of local row 0
    n_total: int = 0                   # global rows of the full table
    meta: dict = field(default_factory=dict)

    def col(self, name: str) -> Column:
        for c in self.columns:
            if c.name == name:
                return c
        raise KeyError(name)

    def index(self, name: str) -> int:
        for i, c in enumerate(self.columns):
            if c.name == name:
                return i
        raise KeyError(name)

    @property
    def types(self) -> list:
        return [c.ctype for c in self.columns]

    def nbytes(self, names=None) -> int:
        cols = self.columns if names is None else [self.col(n) for n in names]
        return sum(c.width * self.n_rows for c in cols)
