"""bench.py's multi-rank plumbing on CPU (gloo, world 2): `--gpus 2` without
a torchrun environment spawns two ranks, C5 items are split without overlap
or gap (no data-path collective), the max-over-ranks reduction works, and
the rank-0 line is labelled with the ranks that actually ran."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _dry(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                               "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--dry-run", *args], capture_output=True,
                       text=True, timeout=600, env=env, cwd=REPO)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


@pytest.mark.slow
def test_c5_two_ranks_split_items():
    line = _dry("--gpus", "2", "--config", "C5", "--items", "8")
    assert line["n_gpus"] == 2 and line["dry_run"] is True
    assert line["scaling"] == "strong" and "batch-shard x2" in line["config"]["parallelism"]
    sh = sorted(line["shards"], key=lambda x: x["rank"])
    assert [x["first_item"] for x in sh] == [0, 4] and [x["items"] for x in sh] == [4, 4]
    assert line["grid_points_per_step_job"] == 8 * 512 * 512
    assert line["max_over_ranks_check"] == 1.0  # max of the ranks' values (0, 1)


def test_shard_items_partition():
    sys.path.insert(0, REPO)
    import bench

    for items, world in ((512, 1), (512, 2), (512, 8), (10, 3)):
        got = [bench.shard_items(items, r, world) for r in range(world)]
        firsts = [f for f, _ in got]
        per = got[0][1]
        assert all(n == per for _, n in got) and per == items // world
        assert firsts == [r * per for r in range(world)]


def test_single_rank_dry_run_c2():
    line = _dry("--config", "C2")
    assert line["n_gpus"] == 1 and line["grid_points_per_step_job"] == 2048 * 2048
    assert "replicas" in line["config"]["parallelism"]


def test_c4_step_bytes_model():
    """The C4 roofline's byte model: the fused-schedule pass model of DESIGN section 4, summed by hand."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    c, M = (1024, 1024, 1024), (2048, 2048, 2048)
    H = M[2] // 2 + 1
    ks = (M[0] // 2 + 1) * (M[1] // 2 + 1) * H * 8
    plane, slab, N = 16 * c[0] * M[1] * H, 16 * c[0] * c[1] * H, c[0] * c[1] * c[2]
    want = (2 * slab + 2 * plane) + 4 * (ks + 2 * plane + 2 * slab + 8 * N)
    want += 3 * (2 * slab + 2 * plane + ks) + 2 * plane + 2 * slab + 9 * N
    got = bench.c4_step_bytes(c, M)
    assert got == want
    # between the compulsory output bytes and SURVEY 8(d)'s looser 1640 B/pt
    assert 41 * N < got < bench.SURVEY_BYTES_PER_POINT["C4"] * N
