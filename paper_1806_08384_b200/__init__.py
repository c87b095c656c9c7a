"""paper_1806_08384_b200 — the exact-selectivity probe of Shin 2018 (arXiv 1806.08384) on B200.

`Table.count(P)` is the paper's `SELECT COUNT(*) FROM R WHERE P` (Listing 3.1)
and `Table.pushdown(P, project)` materialises sigma_P pi_project(R), both on
hand-written sm_100a kernels behind the C ABI of include/sel.h (libsel.so). torch supplies device
memory, streams and process groups only.
"""

from ._native import SelError, EXPORTS
from .predicate import col, TRUE, FALSE, INT32, INT64, FLOAT32, DATE32, DICT8, DICT16, DICT32
from .api import (Context, Table, PushdownResult, ExecuteResult, program_check, program_path,
                  program_plan, equi_depth_estimate)

__all__ = ["SelError", "EXPORTS", "col", "TRUE", "FALSE", "INT32", "INT64", "FLOAT32", "DATE32",
           "DICT8", "DICT16", "DICT32", "Context", "Table", "PushdownResult", "ExecuteResult", "program_check",
           "program_path", "program_plan", "equi_depth_estimate"]
