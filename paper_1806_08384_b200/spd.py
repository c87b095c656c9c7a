"""Algorithm 1 — Selective Selection Push-Down as a host driver over the probe.

    EvaluateAndPushDown(treeRA):
      listRA <- priority queue of scans R with R.size > PUSH_DOWN_MIN_TABLE_SIZE
      listRA.pop()                        # the largest relation is probed, never pushed
      for each R in listRA:
        (conditions, columns) <- ExtractPushDown(R); compound <- CoalesceNodes(...)
        try:   maxSize <- R.size * PUSH_DOWN_MAX_SELECTIVITY
               resultSet <- Execute(compound, true, maxSize)   # count, throw if > maxSize
               AddTemporaryTable(resultSet); UpdateTree(treeRA)
        catch: revert the push-down for R

The plan rewrite itself (ExtractPushDown, CoalesceNodes, AddTemporaryTable, UpdateTree) belongs to a
query compiler and is out of scope: a caller hands each relation's pushed-down
predicate and needed columns in directly, and gets back, per relation, the exact count (what the
optimizer orders joins by) and — if the push-down was kept — the materialised sigma pi(R)
("temporary table"). Execute(compound, isSPD=true, maxSize) is one C-ABI call, `sel_execute`.

Readings: priority ties are broken by relation name; the size filter
is strict ">"; maxSize = floor(R.size * ratio) when PUSH_DOWN_MAX_SELECTIVITY is a ratio,
or the number itself when given as an absolute row count; a relation with no pushed-down
condition has nothing to push and is skipped.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence


@dataclass
class Relation:
    name: str
    size: int                                    # R.size (global rows)
    predicate: object = None                     # pushed-down conditions (ExtractPushDown)
    project: Sequence = ()                       # needed columns (ExtractPushDown)
    table: object = None                         # a registered paper_1806_08384_b200.Table


@dataclass
class Decision:
    name: str
    size: int
    role: str                                    # "probe" | "too_small" | "no_condition" | "evaluated"
    count: Optional[int] = None                  # exact |sigma(R)| when evaluated
    max_size: Optional[int] = None
    pushed: bool = False                         # True: materialised (temp table); False: reverted
    result: object = None                        # ExecuteResult (the temporary table) when pushed

    @property
    def selectivity(self) -> Optional[float]:
        return None if self.count is None or self.size == 0 else self.count / self.size


def max_size_for(size: int, max_selectivity) -> int:
    """PUSH_DOWN_MAX_SELECTIVITY as a ratio (float) or an absolute row count (int)."""
    if isinstance(max_selectivity, float):
        return int(math.floor(size * max_selectivity))
    return int(max_selectivity)


def evaluate_and_push_down(relations: Sequence[Relation], min_table_size: int,
                           max_selectivity, execute: Callable | None = None) -> list:
    """Algorithm 1 over `relations`; returns one Decision per relation in processing order
    (probe first, then the queue in size order, then the filtered ones).

    execute(relation, max_size) -> (count, materialized, result) defaults to the relation's
    Table.execute (Execute(compound, isSPD=true, maxSize) on the GPU)."""
    if execute is None:
        def execute(rel, max_size):
            r = rel.table.execute(rel.predicate, project=list(rel.project), max_size=max_size)
            return r.count, r.materialized, (r if r.materialized else None)
    heap, decisions = [], []
    for rel in relations:
        if rel.size > min_table_size:                                   # P:368 (strict)
            heapq.heappush(heap, (-rel.size, rel.name, rel))
        else:
            decisions.append(Decision(rel.name, rel.size, "too_small"))
    ordered = [heapq.heappop(heap)[2] for _ in range(len(heap))]
    out = []
    if ordered:
        probe = ordered.pop(0)
        out.append(Decision(probe.name, probe.size, "probe"))
    for rel in ordered:
        if rel.predicate is None:
            out.append(Decision(rel.name, rel.size, "no_condition"))
            continue
        ms = max_size_for(rel.size, max_selectivity)
        count, materialized, result = execute(rel, ms)
        out.append(Decision(rel.name, rel.size, "evaluated", count=count, max_size=ms,
                            pushed=bool(materialized), result=result))
    return out + decisions
