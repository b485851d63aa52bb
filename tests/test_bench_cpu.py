"""bench.py's launcher (CPU): --gpus N with WORLD_SIZE unset re-executes
itself under torch.distributed.run with N ranks (the driver's N>1 path)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_bench_spawns_ranks_without_torchrun():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--workload", "ranks"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 for l in lines)


def test_lpt_assignment_balances_the_batch():
    sys.path.insert(0, str(ROOT))
    import bench

    sides = [128, 256, 512]
    costs = [5 * sides[i % 3] ** 3 * 3.0 for i in range(4096)]
    for world in (1, 2, 4, 8):
        owner = bench.lpt_assign(costs, world)
        loads = [sum(c for c, o in zip(costs, owner) if o == r) for r in range(world)]
        assert max(loads) <= (sum(costs) / world) * 1.01
