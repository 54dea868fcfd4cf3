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


# ---- the remaining cases of proj/tests/test_cli.cpp, one to one --------------
def test_unknown_kernel_exits_1():
    """test_cli.cpp:98-101."""
    assert run("bench", "--kernel", "bogus-kernel").returncode == 1
    assert run("verify", "--kernel", "bogus-kernel").returncode == 1


def test_configuration_errors_exit_1_reference_cases():
    """test_cli.cpp:103-115: odd iterations with an AA kernel, bad dims
    syntax, bad geometry kind, bad padding -- all before any device work."""
    for args in (["bench", "--kernel", "aa-soa", "--geometry", "blocks", "--dims", "12x10x10",
                  "--iterations", "5"],
                 ["geometry", "--kind", "channel", "--dims", "chunky"],
                 ["geometry", "--kind", "torus", "--dims", "4x4x4"],
                 ["bench", "--kernel", "list-aa-soa", "--geometry", "blocks", "--dims", "12x10x10",
                  "--iterations", "2", "--padding", "1,2,3"]):
        assert run(*args).returncode == 1, args


@pytest.mark.gpu
def test_geometry_subcommand_emits_fluid_statistics():
    """test_cli.cpp:117-120: blocks 16^3, b = s = 4 -> 3584 fluid nodes."""
    r = run("geometry", "--kind", "blocks", "--dims", "16x16x16", "--block", "4", "--spacing", "4",
            "--stats")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["fluid_nodes"] == 16 ** 3 - 8 * 4 ** 3 and j["periodic"] == [True, True, True]
    assert j["fluid_fraction"] == pytest.approx(1.0 - 0.5 ** 3)


@pytest.mark.gpu
def test_csv_row_and_json_carry_the_same_information():
    """test_cli.cpp:32-59: blocks 12x10x10, list-aa-soa, seed 9: as many
    fields as header columns; kernel, geometry and B_l = 340 in both."""
    args = ["bench", "--kernel", "list-aa-soa", "--geometry", "blocks", "--dims", "12x10x10",
            "--iterations", "10", "--warmup", "2", "--seed", "9"]
    head, row = run(*args).stdout.strip().splitlines()
    js = run(*args, "--format", "json").stdout
    assert head.startswith(REF_COLUMNS) and row.count(",") == head.count(",")
    for token in ("list-aa-soa", "blocks", "340"):
        assert token in row and token in js, token
    rec, j = dict(zip(head.split(","), row.split(","))), json.loads(js)
    assert rec["state_hash"] == j["state_hash"] and int(rec["n_fluid"]) == j["n_fluid"] == 1136


@pytest.mark.gpu
def test_bench_appends_csv_rows_with_one_header(tmp_path):
    """test_cli.cpp:122-140: two runs with --out -> one header, three lines."""
    path = tmp_path / "lbm_cli_test.csv"
    for _ in range(2):
        r = run("bench", "--kernel", "list-aa-soa", "--geometry", "blocks", "--dims", "12x10x10",
                "--iterations", "4", "--warmup", "0", "--threads", "1", "--out", str(path))
        assert r.returncode == 0 and r.stdout == "", r.stderr
    lines = path.read_text().splitlines()
    assert len(lines) == 3
    assert sum(1 for ln in lines if ln.startswith("schema_version")) == 1
    assert lines[1].split(",")[-1] == lines[2].split(",")[-1]  # same state hash both runs


@pytest.mark.gpu
def test_verify_subcommand_exit_codes_reference_case():
    """test_cli.cpp:159-168."""
    assert run("verify", "--kernel", "list-aa-soa", "--dims", "4x4x14", "--interval", "400", "--tol",
               "1e-11").returncode == 0
    assert run("verify", "--kernel", "list-aa-soa", "--dims", "4x4x14", "--interval", "100", "--tol",
               "1e-14", "--max-steps", "200").returncode == 3


def test_microbench_unknown_kind_exits_1():
    """micro_kind_from_string (perfmodel.cpp:59-64): the error lists the kinds."""
    r = run("microbench", "--which", "triad")
    assert r.returncode == 1 and "valid: copy, copy-19, copy-19-nt-sl, update-19" in r.stderr
    assert run("bench", "--kernel", "aa-soa", "--bandwidths", "/nonexistent").returncode == 1


@pytest.mark.gpu
def test_microbench_writes_the_bandwidth_file_bench_reads(tmp_path):
    """cmd_microbench (cli.cpp:333-358) with the device micro-benchmarks:
    `--out` writes the reference's bandwidth-file format (perfmodel.cpp:98-
    128), a second run merges into it, and `bench --bandwidths` takes its
    roofline ceiling from the micro-benchmark that models the kernel."""
    path = tmp_path / "bw.txt"
    r = run("microbench", "--which", "update-19", "--size", str(2 << 30), "--reps", "3", "--out",
            str(path))
    assert r.returncode == 0 and "update-19" in r.stdout, r.stderr
    r = run("microbench", "--which", "copy-19", "--size", str(2 << 30), "--reps", "3", "--out",
            str(path))
    assert r.returncode == 0, r.stderr
    lines = path.read_text().splitlines()
    assert lines[0] == "# micro-benchmark bandwidths [GB/s]"
    bw = {ln.split()[0]: float(ln.split()[1]) for ln in lines[1:]}
    assert set(bw) == {"copy-19", "update-19"} and all(3000 < v < 8000 for v in bw.values())
    r = run("bench", "--kernel", "aa-soa", "--dims", "64x64x64", "--iterations", "10", "--format",
            "json", "--bandwidths", str(path))
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["pmax_mflups"] == pytest.approx(bw["update-19"] * 1000 / 304, rel=1e-5)
