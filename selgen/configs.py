"""Synthetic workloads of BASELINE.json's configs, generated from the master
seed 180608384. Every generator takes a global row range [row_start, row_start + row_count) so
each rank of a sharded run builds exactly its own contiguous shard.

C1  TPC-H lineitem SF-0.01 (60,000 rows), Listing 1.1 mapped onto lineitem, COUNT only.
C2  the paper's worked example R (600M rows): a tuple multiset with exact
    multiplicities scattered by an affine bijection; COUNT + push-down projecting A, C, D.
C3  TPC-H lineitem SF-50 (300M rows) with Q3/Q5/Q10-style predicates.
C4  SSB lineorder SF-80 (480M rows) with Q1.x, Q3.x, Q4.x date/discount/quantity predicates.
C5  1e9-row selectivity sweep: x = (a*i + b) mod N, predicate x < t.

Nothing here evaluates a predicate; the closed-form facts the tests use (tuple lists and
multiplicities, affine parameters) are exposed as table metadata.
"""

from __future__ import annotations

import datetime as _dt
import math

import numpy as np
import torch

from .hashing import derive_seed, h32, splitmix64, uniform_int
from .program import (Cmp, Between, In, InSet, And, Or, Const, INT32, INT64, DATE32, DICT8)
from .tables import Column, Table, to_storage, STORAGE_DTYPE

EPOCH = _dt.date(1970, 1, 1)
DEFAULT_CHUNK = 1 << 25


def date32(y: int, m: int, d: int) -> int:
    """DATE32 = days since 1970-01-01."""
    return (_dt.date(y, m, d) - EPOCH).days


def yyyymmdd(day32: int) -> int:
    d = EPOCH + _dt.timedelta(days=day32)
    return d.year * 10000 + d.month * 100 + d.day


ORDERDATE_LO = date32(1992, 1, 1)           # 8035
ORDERDATE_HI = date32(1998, 8, 2)           # 10440 (2,406 days)
RETURN_CUTOFF = date32(1995, 6, 17)         # 9298
RETURNFLAG_DICT = ["A", "N", "R"]           # sorted dictionary: code order = string order
SHIPMODE_DICT = ["AIR", "FOB", "MAIL", "RAIL", "REG AIR", "SHIP", "TRUCK"]


def _chunks(row_start, row_count, chunk):
    s = row_start
    end = row_start + row_count
    while s < end:
        e = min(end, s + chunk)
        yield s, e
        s = e


def _alloc(ctype, n, device):
    return torch.empty(n, dtype=STORAGE_DTYPE[ctype], device=device)


def choose_affine(n: int, *seed_path) -> tuple:
    """Affine bijection π(j) = (a*j + b) mod n with gcd(a, n) = 1.
    Returns (a, b, a_inv)."""
    assert 0 < n < 3_000_000_000, "a*j must stay below 2^63 in int64"
    if n == 1:
        return 1, 0, 1
    s = derive_seed(*seed_path)
    a = (splitmix64(s) % n) | 1
    while math.gcd(a, n) != 1 or a % 5 == 0:
        a = (a + 2) % n or 1
    b = splitmix64(s ^ 0xB) % n
    return a, b, pow(a, -1, n)


# ------------------------------------------------------------------------------------------
# C2: the worked example, SURVEY §8c "C2 generator, P3 form".

C2_ROWS = 600_000_000
C2_X, C2_Y2, C2_Y1, C2_Z1, C2_Z2 = 2, 1000, 2001, 1, 4
_B_IN = list(range(1001, 2001))                            # y2 < B < y1
_B_OUT = list(range(0, 501)) + list(range(2001, 2500))     # 1,000 values outside (y2, y1)


def c2_groups(n_total: int):
    """Tuple groups (A values, B values, C values, total rows) for R scaled to n_total rows.
    n_total must be a multiple of 6,000 so every group total is an integer."""
    assert n_total % 6000 == 0, "C2 group totals need n_total divisible by 6000"
    f = n_total // 6000                        # 600M -> 100,000
    return [
        ("H",  [C2_X], _B_IN, [C2_Z1, C2_Z2], 1002 * f),            # 100.2M: all four true
        ("M1", [C2_X], _B_IN, [0, 2, 3, 5, 6], 99 * f),             # 9.9M: C fails
        ("M2", [C2_X], _B_OUT, [C2_Z1, C2_Z2], 99 * f),             # 9.9M: B fails
    ] + [  # 480M where A fails, 120M per A value so that every A value holds N/5 rows
        (f"O{a}", [a], _B_IN + _B_OUT, list(range(7)), 1200 * f) for a in (0, 1, 3, 4)
    ]


def c2_tuples(n_total: int):
    """Distinct tuples (A, B, C) with exact multiplicities in source order (numpy int64)."""
    A, B, C, M = [], [], [], []
    for _, avals, bvals, cvals, total in c2_groups(n_total):
        ta, tb, tc = np.meshgrid(np.array(avals), np.array(bvals), np.array(cvals), indexing="ij")
        ta, tb, tc = ta.ravel(), tb.ravel(), tc.ravel()
        k = ta.size
        m = np.full(k, total // k, dtype=np.int64)
        m[: total % k] += 1
        A.append(ta); B.append(tb); C.append(tc); M.append(m)
    return (np.concatenate(A).astype(np.int64), np.concatenate(B).astype(np.int64),
            np.concatenate(C).astype(np.int64), np.concatenate(M))


def gen_c2(n_total: int = C2_ROWS, row_start: int = 0, row_count: int | None = None,
           device="cpu", chunk: int = DEFAULT_CHUNK) -> Table:
    """R(A INT32, B INT32, C DICT8 (7 codes), D INT32 payload)."""
    if row_count is None:
        row_count = n_total - row_start
    ta, tb, tc, tm = c2_tuples(n_total)
    ends = np.cumsum(tm)
    assert int(ends[-1]) == n_total
    a, b, a_inv = choose_affine(n_total, "C2", "pi")
    d_seed = derive_seed("C2", "D")
    dev = torch.device(device)
    t_a = torch.from_numpy(ta).to(dev)
    t_b = torch.from_numpy(tb).to(dev)
    t_c = torch.from_numpy(tc).to(dev)
    t_end = torch.from_numpy(ends).to(dev)
    A = _alloc(INT32, row_count, dev)
    B = _alloc(INT32, row_count, dev)
    C = _alloc(DICT8, row_count, dev)
    D = _alloc(INT32, row_count, dev)
    for s, e in _chunks(row_start, row_count, chunk):
        i = torch.arange(s, e, dtype=torch.int64, device=dev)
        j = (a_inv * ((i - b) % n_total)) % n_total        # source position: π(j) = i
        k = torch.searchsorted(t_end, j, right=True)
        o, p = s - row_start, e - row_start
        A[o:p] = t_a[k].to(torch.int32)
        B[o:p] = t_b[k].to(torch.int32)
        C[o:p] = t_c[k].to(torch.uint8)
        D[o:p] = to_storage(h32(d_seed, i) - (1 << 31), INT32)
    cols = [Column("A", INT32, A), Column("B", INT32, B), Column("C", DICT8, C, 7),
            Column("D", INT32, D)]
    return Table("C2", cols, row_count, row_start, n_total,
                 meta={"affine": (a, b, a_inv), "tuples": (ta, tb, tc, tm), "d_seed": d_seed})


def c2_probes():
    """Listing 3.1 in three encodings; columns A0 B1 C2."""
    A, B, C = 0, 1, 2
    lit = And(And(And(Cmp("=", A, C2_X), Cmp("<", B, C2_Y1)), Cmp(">", B, C2_Y2)),
              Or(Cmp("=", C, C2_Z1), Cmp("=", C, C2_Z2)))
    between_in = And(And(Cmp("=", A, C2_X), Between(B, C2_Y2 + 1, C2_Y1 - 1)),
                     In(C, (C2_Z1, C2_Z2)))
    between_or = And(And(Cmp("=", A, C2_X), Between(B, C2_Y2 + 1, C2_Y1 - 1)),
                     Or(Cmp("=", C, C2_Z1), Cmp("=", C, C2_Z2)))
    return {"listing": lit, "between_in": between_in, "between_or": between_or}


C2_PROJECT = [0, 2, 3]          # A, C, D ("column A ... C and D")


# ------------------------------------------------------------------------------------------
# C1 / C3: TPC-H lineitem-shaped (dbgen-like rules; external convention).

LINEITEM_COLS = ["l_orderkey", "l_quantity", "l_discount", "l_extendedprice",
                 "l_returnflag", "l_shipdate", "l_receiptdate", "l_shipmode"]


def gen_lineitem(n_total: int, row_start: int = 0, row_count: int | None = None, device="cpu",
                 columns=None, chunk: int = DEFAULT_CHUNK) -> Table:
    if row_count is None:
        row_count = n_total - row_start
    names = LINEITEM_COLS if columns is None else [c for c in LINEITEM_COLS if c in columns]
    types = {"l_orderkey": INT32, "l_quantity": INT32, "l_discount": INT32,
             "l_extendedprice": INT64, "l_returnflag": DICT8, "l_shipdate": DATE32,
             "l_receiptdate": DATE32, "l_shipmode": DICT8}
    dsz = {"l_returnflag": 3, "l_shipmode": 7}
    dev = torch.device(device)
    out = {n: _alloc(types[n], row_count, dev) for n in names}
    sd = {n: derive_seed("lineitem", n) for n in LINEITEM_COLS}
    for s, e in _chunks(row_start, row_count, chunk):
        i = torch.arange(s, e, dtype=torch.int64, device=dev)
        order = i >> 2                                          # ~4 lines per order
        o, p = s - row_start, e - row_start
        odate = uniform_int(sd["l_orderkey"] ^ 0x0D, order, ORDERDATE_LO, ORDERDATE_HI)
        ship = odate + uniform_int(sd["l_shipdate"], i, 1, 121)
        receipt = ship + uniform_int(sd["l_receiptdate"], i, 1, 30)
        if "l_orderkey" in out:
            out["l_orderkey"][o:p] = (order + 1).to(torch.int32)
        if "l_quantity" in out or "l_extendedprice" in out:
            qty = uniform_int(sd["l_quantity"], i, 1, 50)
            if "l_quantity" in out:
                out["l_quantity"][o:p] = qty.to(torch.int32)
            if "l_extendedprice" in out:
                out["l_extendedprice"][o:p] = qty * uniform_int(sd["l_extendedprice"], i, 90_000, 200_000)
        if "l_discount" in out:
            out["l_discount"][o:p] = uniform_int(sd["l_discount"], i, 0, 10).to(torch.int32)
        if "l_returnflag" in out:
            ra = uniform_int(sd["l_returnflag"], i, 0, 1) * 2          # 'A'=0 or 'R'=2
            out["l_returnflag"][o:p] = torch.where(receipt <= RETURN_CUTOFF, ra,
                                                   torch.ones_like(ra)).to(torch.uint8)
        if "l_shipdate" in out:
            out["l_shipdate"][o:p] = ship.to(torch.int32)
        if "l_receiptdate" in out:
            out["l_receiptdate"][o:p] = receipt.to(torch.int32)
        if "l_shipmode" in out:
            out["l_shipmode"][o:p] = uniform_int(sd["l_shipmode"], i, 0, 6).to(torch.uint8)
    cols = [Column(n, types[n], out[n], dsz.get(n, 0)) for n in names]
    return Table("lineitem", cols, row_count, row_start, n_total)


def lineitem_probes(table: Table):
    """Predicates of SURVEY §8d C1/C3 on lineitem columns (indices resolved by name)."""
    ix = table.index
    R, MAIL, SHIP = RETURNFLAG_DICT.index("R"), SHIPMODE_DICT.index("MAIL"), SHIPMODE_DICT.index("SHIP")
    probes = {}
    try:
        rf, sd, sm = ix("l_returnflag"), ix("l_shipdate"), ix("l_shipmode")
        # Listing 1.1 mapped: A->returnflag, B->shipdate (1994), C->shipmode
        probes["listing1"] = And(And(And(Cmp("=", rf, R), Cmp(">", sd, date32(1994, 1, 1))),
                                     Cmp("<", sd, date32(1995, 1, 1))),
                                 Or(Cmp("=", sm, MAIL), Cmp("=", sm, SHIP)))
    except KeyError:
        pass
    try:
        sd = ix("l_shipdate")
        probes["q3"] = Cmp(">", sd, date32(1992, 2, 1))
        probes["q5"] = And(Cmp(">=", sd, date32(1993, 1, 1)), Cmp("<", sd, date32(1994, 1, 1)))
        rf = ix("l_returnflag")
        probes["q10"] = And(And(Cmp(">=", sd, date32(1993, 7, 1)), Cmp("<", sd, date32(1993, 10, 1))),
                            Cmp("=", rf, R))
    except KeyError:
        pass
    return probes


# ------------------------------------------------------------------------------------------
# C4: SSB lineorder-shaped (SSB convention 6M x SF rows).

LINEORDER_COLS = ["lo_orderdate", "lo_discount", "lo_quantity", "lo_revenue"]


def _datekeys(device):
    keys = [yyyymmdd(d) for d in range(ORDERDATE_LO, ORDERDATE_HI + 1)]
    return torch.tensor(keys, dtype=torch.int64, device=device)


def gen_lineorder(n_total: int, row_start: int = 0, row_count: int | None = None, device="cpu",
                  chunk: int = DEFAULT_CHUNK) -> Table:
    if row_count is None:
        row_count = n_total - row_start
    dev = torch.device(device)
    keys = _datekeys(dev)
    out = {n: _alloc(INT32, row_count, dev) for n in LINEORDER_COLS}
    sd = {n: derive_seed("lineorder", n) for n in LINEORDER_COLS}
    for s, e in _chunks(row_start, row_count, chunk):
        i = torch.arange(s, e, dtype=torch.int64, device=dev)
        o, p = s - row_start, e - row_start
        out["lo_orderdate"][o:p] = keys[uniform_int(sd["lo_orderdate"], i >> 2, 0, keys.numel() - 1)].to(torch.int32)
        out["lo_discount"][o:p] = uniform_int(sd["lo_discount"], i, 0, 10).to(torch.int32)
        out["lo_quantity"][o:p] = uniform_int(sd["lo_quantity"], i, 1, 50).to(torch.int32)
        out["lo_revenue"][o:p] = uniform_int(sd["lo_revenue"], i, 100, 10_000_000).to(torch.int32)
    cols = [Column(n, INT32, out[n]) for n in LINEORDER_COLS]
    return Table("lineorder", cols, row_count, row_start, n_total)


def lineorder_probes():
    od, disc, qty = 0, 1, 2
    return {
        "q1.1": And(And(Between(od, 19930101, 19931231), Between(disc, 1, 3)), Cmp("<", qty, 25)),
        "q1.2": And(And(Between(od, 19940101, 19940131), Between(disc, 4, 6)), Between(qty, 26, 35)),
        "q1.3": And(And(Between(od, 19940205, 19940211), Between(disc, 5, 7)), Between(qty, 26, 35)),
        "q3.1": Between(od, 19920101, 19971231),
        "q3.4": Between(od, 19971201, 19971231),
        "q4.2": Or(Between(od, 19970101, 19971231), Between(od, 19980101, 19981231)),
    }


# ------------------------------------------------------------------------------------------
# C6: SSB Q2.x-shaped semijoin probes. The paper's SSB
# queries use integer-coded dimension attributes (p_category = 12, s_region = 1, p_brand1 in
# 2221..2228). Dimension sizes follow the SSB convention: part 200,000 x floor(1 + log2 SF),
# supplier 2,000 x SF. p_category = mfgr*10 + category (mfgr, category in 1..5), p_brand1 =
# p_category*100 + brand (brand in 1..40), s_region in 0..4, all by seeded hash of the key.
# The dimension selections become key sets over lo_partkey / lo_suppkey (the fact-table probe is
# the hot path; building the sets is the join side, out of scope, done here as input prep).

LINEORDER_Q2_COLS = ["lo_orderdate", "lo_partkey", "lo_suppkey", "lo_revenue"]


def ssb_sizes(sf: int) -> dict:
    return {"lineorder": 6_000_000 * sf, "part": 200_000 * int(math.floor(1 + math.log2(sf))),
            "supplier": 2_000 * sf}


def gen_lineorder_q2(n_total: int, sf: int, row_start: int = 0, row_count: int | None = None,
                     device="cpu", chunk: int = DEFAULT_CHUNK) -> Table:
    if row_count is None:
        row_count = n_total - row_start
    dev = torch.device(device)
    keys = _datekeys(dev)
    sz = ssb_sizes(sf)
    out = {n: _alloc(INT32, row_count, dev) for n in LINEORDER_Q2_COLS}
    sd = {n: derive_seed("lineorder_q2", n) for n in LINEORDER_Q2_COLS}
    for s, e in _chunks(row_start, row_count, chunk):
        i = torch.arange(s, e, dtype=torch.int64, device=dev)
        o, p = s - row_start, e - row_start
        out["lo_orderdate"][o:p] = keys[uniform_int(sd["lo_orderdate"], i >> 2, 0, keys.numel() - 1)].to(torch.int32)
        out["lo_partkey"][o:p] = uniform_int(sd["lo_partkey"], i, 1, sz["part"]).to(torch.int32)
        out["lo_suppkey"][o:p] = uniform_int(sd["lo_suppkey"], i, 1, sz["supplier"]).to(torch.int32)
        out["lo_revenue"][o:p] = uniform_int(sd["lo_revenue"], i, 100, 10_000_000).to(torch.int32)
    cols = [Column(n, INT32, out[n]) for n in LINEORDER_Q2_COLS]
    return Table("lineorder_q2", cols, row_count, row_start, n_total)


def ssb_dimensions(sf: int) -> dict:
    """Integer-coded dimension attributes indexed by key (index 0 unused): p_category, p_brand1,
    s_region (numpy int64)."""
    sz = ssb_sizes(sf)
    pk = torch.arange(sz["part"] + 1, dtype=torch.int64)
    sk = torch.arange(sz["supplier"] + 1, dtype=torch.int64)
    mfgr = uniform_int(derive_seed("part", "mfgr"), pk, 1, 5)
    cat = uniform_int(derive_seed("part", "category"), pk, 1, 5)
    brand = uniform_int(derive_seed("part", "brand"), pk, 1, 40)
    p_category = mfgr * 10 + cat
    return {"p_category": p_category.numpy(), "p_brand1": (p_category * 100 + brand).numpy(),
            "s_region": uniform_int(derive_seed("supplier", "region"), sk, 0, 4).numpy()}


def key_set(mask: np.ndarray) -> tuple:
    """(uint64 words, nbits) of the keys k with mask[k] (k = 0 .. len(mask)-1)."""
    nb = len(mask)
    bits = np.zeros(((nb + 63) // 64) * 64, dtype=np.uint8)
    bits[:nb] = mask[:nb] != 0
    bits[0] = 0                                                   # key 0 is not a key
    return np.packbits(bits, bitorder="little").view(np.uint64).copy(), nb


def q2_probes(sf: int):
    """{name: (AST over LINEORDER_Q2_COLS with key-set ids 0 and 1, [part set, supplier set])}
    for SSB Q2.1-Q2.3."""
    dims = ssb_dimensions(sf)
    pc, pb, sr = dims["p_category"], dims["p_brand1"], dims["s_region"]
    node = And(InSet(1, 0), InSet(2, 1))
    return {
        "q2.1": (node, [key_set(pc == 12), key_set(sr == 1)]),
        "q2.2": (node, [key_set((pb >= 2221) & (pb <= 2228)), key_set(sr == 2)]),
        "q2.3": (node, [key_set(pb == 2239), key_set(sr == 3)]),
    }


# ------------------------------------------------------------------------------------------
# C5: selectivity sweep on an affine-threshold column.

C5_ROWS = 1_000_000_000
C5_SELECTIVITIES = [1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 0.1, 0.5, 1.0]


def gen_sweep(n_total: int = C5_ROWS, row_start: int = 0, row_count: int | None = None,
              device="cpu", layout: str = "scattered", chunk: int = DEFAULT_CHUNK) -> Table:
    """x INT32 = (a*i + b) mod N ("scattered") or x = i ("clustered"); y INT32 payload."""
    if row_count is None:
        row_count = n_total - row_start
    dev = torch.device(device)
    a, b, a_inv = choose_affine(n_total, "C5", "x")
    y_seed = derive_seed("C5", "y")
    X = _alloc(INT32, row_count, dev)
    Y = _alloc(INT32, row_count, dev)
    for s, e in _chunks(row_start, row_count, chunk):
        i = torch.arange(s, e, dtype=torch.int64, device=dev)
        o, p = s - row_start, e - row_start
        X[o:p] = ((a * i + b) % n_total if layout == "scattered" else i).to(torch.int32)
        Y[o:p] = to_storage(h32(y_seed, i) - (1 << 31), INT32)
    return Table("sweep", [Column("x", INT32, X), Column("y", INT32, Y)], row_count, row_start,
                 n_total, meta={"affine": (a, b, a_inv), "layout": layout})


def sweep_threshold(n_total: int, s: float) -> int:
    return int(round(s * n_total))


def sweep_probe(t: int):
    return Cmp("<", 0, t)


# ------------------------------------------------------------------------------------------
# C0 (optional context workload): TPC-H orders-shaped, for the paper's own probes
# Listings 5.1-5.3.

ORDERSTATUS_DICT = ["F", "O", "P"]
ORDERS_COLS = ["o_orderkey", "o_custkey", "o_orderstatus", "o_totalprice", "o_orderdate"]


def orders_key(i: torch.Tensor) -> torch.Tensor:
    """TPC-H sparse order keys: of every 32 keys only the first 8 are used (distinct, >= 1)."""
    return (i >> 3) * 32 + (i & 7) + 1


def gen_orders(n_total: int, row_start: int = 0, row_count: int | None = None, device="cpu",
               chunk: int = DEFAULT_CHUNK) -> Table:
    if row_count is None:
        row_count = n_total - row_start
    dev = torch.device(device)
    sd = {n: derive_seed("orders", n) for n in ORDERS_COLS}
    types = {"o_orderkey": INT32, "o_custkey": INT32, "o_orderstatus": DICT8,
             "o_totalprice": INT64, "o_orderdate": DATE32}
    out = {n: _alloc(types[n], row_count, dev) for n in ORDERS_COLS}
    n_cust = max(1, n_total // 10)
    for s, e in _chunks(row_start, row_count, chunk):
        i = torch.arange(s, e, dtype=torch.int64, device=dev)
        o, p = s - row_start, e - row_start
        out["o_orderkey"][o:p] = orders_key(i).to(torch.int32)
        out["o_custkey"][o:p] = uniform_int(sd["o_custkey"], i, 1, n_cust).to(torch.int32)
        out["o_orderstatus"][o:p] = uniform_int(sd["o_orderstatus"], i, 0, 2).to(torch.uint8)
        out["o_totalprice"][o:p] = uniform_int(sd["o_totalprice"], i, 85_000, 55_000_000)
        out["o_orderdate"][o:p] = uniform_int(sd["o_orderdate"], i, ORDERDATE_LO, ORDERDATE_HI).to(torch.int32)
    dsz = {"o_orderstatus": 3}
    cols = [Column(n, types[n], out[n], dsz.get(n, 0)) for n in ORDERS_COLS]
    return Table("orders", cols, row_count, row_start, n_total)


def orders_probes():
    """Listings 5.1, 5.2 and the Listing 5.3 attribute sweep;
    DECIMAL 218611.01 as cents 21861101."""
    k, cu, st, tp, od = 0, 1, 2, 3, 4
    O = ORDERSTATUS_DICT.index("O")
    a1 = Cmp("=", k, 1)
    a2 = And(a1, Cmp("=", cu, 184500))
    a3 = And(a2, Cmp("=", st, O))
    a4 = And(a3, Cmp("=", tp, 21861101))
    return {"l5.1": a1, "l5.2": Cmp(">=", k, 1), "attr1": a1, "attr2": a2, "attr3": a3,
            "attr4": a4,
            "q5_orderdate": And(Cmp(">=", od, date32(1993, 1, 1)), Cmp("<", od, date32(1994, 1, 1)))}
