"""Exhaustive pin of the device's f32 exp over every float input.

The reference computes f32(math.exp(x)) (tensorlite core.py:509; CPython's
math.exp is glibc's exp). The device computes b2::exp_f32 (fexp.cuh):
* CPU: the same formula restated in C (scripts/exp_glibc_check.c, identical
  IEEE double operations) equals f32(glibc exp) on all 2^32 inputs;
* GPU: the device function equals f32(libdevice exp(double x)) on all 2^32
  inputs (scripts/exp_exhaustive.cu); any disagreement would be listed and
  settled against glibc by scripts/exp_exhaustive_check.py.
"""
import json
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FEXP = os.path.join(ROOT, "paper_2602_00125_b200", "csrc", "fexp.cuh")


def _table_inc(dst_dir):
    s = open(FEXP).read()
    start = s.index("kExp2Tab[64] = {") + len("kExp2Tab[64] = {")
    body = s[start:s.index("};", start)]
    assert len(re.findall(r"0x1\.[0-9a-f]+p[+-]\d+", body)) == 64
    with open(os.path.join(dst_dir, "exp_table.inc"), "w") as f:
        f.write(body.strip() + "\n")


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_exp_formula_matches_glibc_on_every_float(tmp_path):
    _table_inc(tmp_path)
    exe = tmp_path / "exp_glibc_check"
    subprocess.run(["gcc", "-O2", "-fopenmp", "-I", str(tmp_path), "-o", str(exe),
                    os.path.join(ROOT, "scripts", "exp_glibc_check.c"), "-lm"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    res = json.loads(out.stdout)
    assert res["inputs"] == 1 << 32
    assert res["mismatches_vs_glibc"] == 0, res


@pytest.mark.gpu
def test_device_exp_matches_libdevice_on_every_float(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "exp_exhaustive"
    subprocess.run([nvcc, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-I", os.path.join(ROOT, "paper_2602_00125_b200", "csrc"), "-o", str(exe),
                    os.path.join(ROOT, "scripts", "exp_exhaustive.cu")], check=True)
    new, v0 = tmp_path / "new.bin", tmp_path / "v0.bin"
    out = subprocess.run([str(exe), str(new), str(v0)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    # every disagreement with libdevice must settle in the device's favour against glibc
    res = subprocess.run(["python", os.path.join(ROOT, "scripts", "exp_exhaustive_check.py"), str(new)],
                         capture_output=True, text=True, check=True)
    for r in json.loads(res.stdout):
        assert r["device_wrong"] == 0, r
