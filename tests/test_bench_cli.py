"""bench.py launch logic and the reference arm, on CPU.

* `--gpus N` without a torchrun environment re-launches itself under
  torch.distributed.run with N ranks (the driver's scaling runs use torchrun
  directly); the hidden --dry-run reports each rank's place without a GPU.
* `--impl reference` times the unmodified reference (oracle/_ref) with the
  same metric and `config` object as our arm, and never loads the product
  package or its CUDA library.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_gpus_flag_spawns_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run", "--config", "C5"], capture_output=True, text=True,
                         timeout=300, env=_env(), cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    # the two ranks share stdout: their lines may interleave, so decode every
    # JSON object in the stream rather than line by line
    dec, text, lines, pos = json.JSONDecoder(), out.stdout, [], 0
    while True:
        pos = text.find("{", pos)
        if pos < 0:
            break
        obj, pos = dec.raw_decode(text, pos)
        lines.append(obj)
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 for l in lines)
    assert lines[0]["config"]["natoms_total"] == 2 * 262144


def test_reference_arm_is_the_reference_only():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    code = (
        "import runpy, sys, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '2', '--warmup', '3']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'product_imported': 'paper_2011_12875_b200' in sys.modules,\n"
        "                  'libsnapgpu': 'libsnapgpu' in maps, 'libsnapref': 'libsnapref' in maps}))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, env=_env(), cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    # the two ranks share stdout: their lines may interleave, so decode every
    # JSON object in the stream rather than line by line
    dec, text, lines, pos = json.JSONDecoder(), out.stdout, [], 0
    while True:
        pos = text.find("{", pos)
        if pos < 0:
            break
        obj, pos = dec.raw_decode(text, pos)
        lines.append(obj)
    line, probe = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0
    assert not probe["product_imported"] and not probe["libsnapgpu"] and probe["libsnapref"]
    sys.path.insert(0, ROOT)
    import argparse

    import bench

    ours = bench.workload_config(argparse.Namespace(config="C2"), 1)
    assert line["config"] == ours
    assert line["cpu_baseline"]["cpu_model"] and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["v1_det_katom_steps_s"] > 0
