"""The lbmbench-gpu CLI (tools/lbmbench_gpu.cpp over include/lbmgpu.hpp):
subcommands, CSV schema and exit codes of the reference CLI
(src/cli.cpp:120-142,406-576; tests/test_cli.cpp)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1711_11468_b200", "bin", "lbmbench-gpu")
REF_COLUMNS = ("schema_version,timestamp,kernel,geometry,nx,ny,nz,blk,padding_mode,threads,"
               "iterations,n_fluid,seconds,mflups,bl_theoretical,pmax_mflups,v_fraction,"
               "nt_streams_effective,affinity_applied")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_list_kernels():
    r = run("list-kernels")
    assert r.returncode == 0 and len(r.stdout.split()) == 17
    # the perf-model report (reference cli.cpp "model") is out of scope here
    assert run("model").returncode == 1


def test_config_errors_exit_1():
    for args in (["bench", "--kernel", "nope"], ["bench", "--kernel", "aa-soa", "--iterations", "3"],
                 ["bench", "--kernel", "aa-soa", "--dims", "8x8"], ["frobnicate"],
                 ["bench", "--kernel", "aa-soa", "--padding", "1,2"],
                 ["bench", "--kernel", "aa-soa", "--tau", "0.4"]):
        r = run(*args)
        assert r.returncode == 1, (args, r.stderr)
        assert "configuration error" in r.stderr


@pytest.mark.gpu
def test_bench_csv_and_json():
    r = run("bench", "--kernel", "list-aa-soa", "--geometry", "blocks", "--dims", "40x40x40",
            "--block", "8", "--spacing", "8", "--iterations", "20", "--warmup", "2")
    assert r.returncode == 0, r.stderr
    head, row = r.stdout.strip().splitlines()
    assert head.startswith(REF_COLUMNS)
    rec = dict(zip(head.split(","), row.split(",")))
    # blocks 40^3, b = s = 8: solid cubes where all three coords % 16 >= 8
    solid = sum(1 for x in range(40) for y in range(40) for z in range(40)
                if x % 16 >= 8 and y % 16 >= 8 and z % 16 >= 8)
    assert rec["kernel"] == "list-aa-soa" and int(rec["n_fluid"]) == 40 ** 3 - solid
    assert float(rec["mflups"]) > 0 and len(rec["state_hash"]) == 16
    r = run("bench", "--kernel", "aa-soa", "--dims", "64x64x64", "--iterations", "10",
            "--format", "json", "--gx", "1e-5", "--tau", "1.0")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["n_fluid"] == 246016 and j["gpu_bytes_per_flup"] == 304.0


@pytest.mark.gpu
def test_bench_state_hash_matches_reference_golden():
    """cfg 1 through the CLI: channel 64^3 blk-push-soa, 100 steps after 0
    warmup -> the reference fingerprint 0fc9230302c2fb25."""
    r = run("bench", "--kernel", "blk-push-soa", "--dims", "64x64x64", "--iterations", "100",
            "--warmup", "0", "--tau", "1.0", "--gx", "1e-5")
    assert r.returncode == 0, r.stderr
    head, row = r.stdout.strip().splitlines()
    rec = dict(zip(head.split(","), row.split(",")))
    assert rec["state_hash"] == "0fc9230302c2fb25"


@pytest.mark.gpu
def test_verify_exit_codes():
    r = run("verify", "--kernel", "list-pull-soa", "--dims", "4x4x18")
    assert r.returncode == 0, r.stdout + r.stderr
    j = json.loads(r.stdout)
    assert j["passed"] and j["converged"] and j["linf_rel"] < 1e-4
    # too few steps to converge -> not passed -> exit 3 (cli.cpp:330)
    r = run("verify", "--kernel", "aa-soa", "--dims", "4x4x18", "--max-steps", "4", "--interval", "2")
    assert r.returncode == 3
