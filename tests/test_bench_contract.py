"""bench.py's launcher contract (no GPU needed): one process per GPU, a
WORLD_SIZE that disagrees with --gpus fails loudly, and both arms print the
same `config` dict."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr


def test_both_arms_share_the_config_dict():
    sys.path.insert(0, ROOT)
    import bench
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert src.count('"config": config_dict(') == 2      # ours and --impl reference
    c = bench.config_dict(256, 4)
    assert c["gates_per_gpu"] == 256 and c["parallelism"].startswith("dp4") and "l2" in c
