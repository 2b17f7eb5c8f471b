"""bench.py contract checks that run without a GPU: the reference arm's JSON
line (keys, units, e2e shape) on a small config, and the sweep/report tools."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "torus2x4", "--m", "65536", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["recv_ok"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["steps"] == 2 and d["warmup"] >= 3     # warm-up is clamped to >= 3


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--config", "torus2x4", "--m", "4096", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and not [x for x in out.stdout.splitlines() if x.startswith("{")]


def test_report_tool(tmp_path):
    src = os.path.join(ROOT, "profiles", "r01_final_scaling_G124.jsonl")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "report.py"), src],
                         capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and "| gk8_2 |" in out.stdout


def test_bound_terms():
    """bench.bound_terms: the north-star bound and the HBM term of a multi-GPU
    run, from the plan's per-GPU bytes (no GPU needed)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.executor import Plan
    from paper_2309_13541_b200.graphs import distance_sum
    hbm = 6538.9
    a = load_artifact("gk8_2")
    m = 16 << 20
    with Plan(a.g, a.sched, m=m, n_gpus=1) as p:
        bt = bench.bound_terms([p.gpu_info(0)], 8, m, distance_sum(a.g), hbm)
    # one GPU: Sigma dist = 118 (BFS) vs 122 chunk-hops of the schedule + self shards
    assert abs(bt["t_lb"] - 2 * m * 118 / (hbm * 1e9)) < 1e-12
    assert bt["hbm_bytes"] == 4362010624 and bt["t_both"] == bt["t_hbm"]   # = the ncu-checked bytes
    a = load_artifact("torus4x4x4")
    m = 4 << 20
    with Plan(a.g, a.sched, m=m, n_gpus=2) as p:
        infos = [p.gpu_info(g) for g in range(2)]
    bt = bench.bound_terms(infos, 64, m, distance_sum(a.g), hbm)
    # 2 GPUs: 32 nodes each; local hops dominate, the HBM term exceeds the NVLink term
    assert bt["nvlink_bytes"] == max(max(i["egress_bytes"], i["ingress_bytes"]) for i in infos)
    assert bt["t_hbm"] > bt["t_lb"] and bt["t_both"] == bt["t_hbm"]


def test_balanced_lowering_option():
    """--lowering balanced: the artifact is re-lowered for the placement of
    --gpus (same ops up to their steps), the workload says so, and the
    reference arm replays that schedule bit-exact."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    a = load_artifact("gk8_2")
    b, gpu = bench.balanced_artifact(a, 1 << 20, 8, "optimized")
    assert sorted(gpu) == list(range(8))
    # the same hops carrying the same chunks (a route's chunk range may be cut into
    # pieces that start at different steps), different steps
    def hops(s):
        cover = {}
        for i in s.instructions:
            cover.setdefault((i.src, i.dst, i.s, i.d), []).append((i.c0, i.c1))
        out = {}
        for k, iv in cover.items():
            iv.sort()
            merged = [list(iv[0])]
            for c0, c1 in iv[1:]:
                assert c0 >= merged[-1][1]                 # no chunk twice on a hop
                if c0 == merged[-1][1]:
                    merged[-1][1] = c1
                else:
                    merged.append([c0, c1])
            out[k] = merged
        return out
    assert hops(b.sched) == hops(a.sched)
    assert [i.t for i in b.sched.instructions] != [i.t for i in a.sched.instructions]
    assert b.meta["balanced"]["step_sync_bytes"] <= 320 << 20
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "8", "--lowering", "balanced", "--m", "4099", "--steps", "2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert "balance" in d["cpu_baseline"]["sample"] and d["cpu_baseline"]["recv_ok"] is True


def test_reference_arm_loads_no_product_library():
    """The reference arm times only the CPU restatement: the product's
    _a2a_exec.so must not be mapped in that process."""
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'gk8_2', '--m', '4096',"
            " '--steps', '1']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('PRODUCT' if '_a2a_exec' in maps else 'CLEAN')\n"
            "print('ORACLE' if 'liboracle_replay' in maps else 'NO-ORACLE')\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "CLEAN" in out.stdout and "ORACLE" in out.stdout


def test_config_identical_in_both_arms():
    """`config` holds only the workload: the reference arm's line carries the
    dict our arm builds with the same function for the same artifact."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "4", "--config", "gk8_2", "--m", "65536", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=dict(os.environ, RANK="0", WORLD_SIZE="4", LOCAL_RANK="0"))
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert d["config"] == bench.config_of("gk8_2", load_artifact("gk8_2"), 65536, 4)
    assert d["config"]["copy_self"] is False and "l2" in d["config"]


def test_autotune_candidates():
    """Three unit orders plus chains for every size; LL up to 1 MiB (16-CTA LL up
    to 64 KiB), LL128 up to 4 MiB."""
    sys.path.insert(0, ROOT)
    import bench
    big = bench.default_candidates(4, 16 << 20)
    assert big == ("static", "cp:1048576", "spread:1048576", "chain:262144")
    assert bench.default_candidates(1, 16 << 20)[2] == "mix:1048576"
    small = bench.default_candidates(2, 4096)
    assert "ll" in small and "ll@16" in small and "ll128" in small
    mid = bench.default_candidates(2, 4 << 20)
    assert "ll128" in mid and "ll" not in mid and "mix:262144" in mid
    assert "spread:262144" in bench.default_candidates(4, 4 << 20)
    assert bench.spec_ctas("ll@16") == ("ll", 16) and bench.spec_ctas("cp:1048576", 7) == ("cp:1048576", 7)


def test_traffic_capture_matches_schedule():
    """A chain run is never reported with the unit queues' DRAM capture."""
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
        tr = json.load(fh)
    chain = tr["gk8_2:16777216:G1:chain:262144"]
    generic = tr["gk8_2:16777216:G1"]
    assert chain["per_launch_bytes"] < generic["per_launch_bytes"]
    assert chain["dram_read_bytes"] < 0.5 * generic["dram_read_bytes"]   # forwarded chunks come from L2
