"""The seeded generators produce byte-identical columns on the CPU and on the GPU (SURVEY §8(d)
timing protocol: "tables are generated on the GPU, hashed, and compared with the CPU
generator's hash on <= 10^8-row slices"). Every GPU-side full-size parity check that uses a
closed form or CPU oracle rests on this. Slices sit deep into each full-size table (large row
indices exercise the hash's 64-bit intermediates) and have ragged lengths."""

import hashlib

import pytest
import torch

from selgen import configs

pytestmark = pytest.mark.gpu

N_SLICE = 3_000_017


def _digest(table):
    h = hashlib.sha256()
    for c in table.columns:
        h.update(c.name.encode())
        h.update(c.data.contiguous().cpu().numpy().tobytes())
    return h.hexdigest()


CASES = {
    "c2": lambda s, n, d: configs.gen_c2(configs.C2_ROWS, s, n, device=d),
    "lineitem": lambda s, n, d: configs.gen_lineitem(300_000_000, s, n, device=d),
    "lineorder": lambda s, n, d: configs.gen_lineorder(480_000_000, s, n, device=d),
    "lineorder_q2": lambda s, n, d: configs.gen_lineorder_q2(480_000_000, 80, s, n, device=d),
    "sweep": lambda s, n, d: configs.gen_sweep(configs.C5_ROWS, s, n, device=d),
    "orders": lambda s, n, d: configs.gen_orders(75_000_000, s, n, device=d),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_cpu_and_gpu_generators_agree(name, cuda_device):
    gen = CASES[name]
    total = {"c2": configs.C2_ROWS, "lineitem": 300_000_000, "lineorder": 480_000_000,
             "lineorder_q2": 480_000_000, "sweep": configs.C5_ROWS, "orders": 75_000_000}[name]
    for start in (0, total // 2 + 12_345, total - N_SLICE):
        cpu = gen(start, N_SLICE, "cpu")
        gpu = gen(start, N_SLICE, cuda_device)
        torch.cuda.synchronize()
        assert _digest(cpu) == _digest(gpu), (name, start)
