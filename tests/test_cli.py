"""The command-line workbench (paper_0810_3203_b200/cli/cftft_cli.cpp) driven
through a pipe, as the reference's cli_test.cpp:22-136 drives its CLI: CSV
headers and shapes, bounds, exit codes, determinism of the non-timing
columns, --inject-fault making verify fail."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def cli():
    from paper_0810_3203_b200._build import build_cli, build_library

    build_library()
    return build_cli()


def run(cli, args):
    r = subprocess.run([cli] + args.split(), capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout


def tft_bound(L, n):
    ell = L.bit_length() - 1
    return min((n - 1) * ell + 2 * (L - 1), L * ell) // 2


def test_count_csv_shape_and_bounds(cli):  # cli_test.cpp:52-70
    rc, out = run(cli, "count --length 8")
    assert rc == 0
    lines = out.splitlines()
    assert len(lines) == 9
    assert lines[0] == "n,tft_count,tft_bound,itft_count,itft_bound"
    for n in range(1, 9):
        f = lines[n].split(",")
        assert len(f) == 5 and int(f[0]) == n
        assert int(f[1]) <= int(f[2]) and int(f[3]) <= int(f[4])
        assert int(f[2]) == tft_bound(8, n) and int(f[4]) == tft_bound(8, n)
    assert lines[8].split(",")[1] == "12" and lines[8].split(",")[3] == "12"


def test_count_policy_flag_and_bad_length(cli):  # cli_test.cpp:72-77
    assert run(cli, "count --length 16 --policy radix2")[0] == 0
    assert run(cli, "count --length 12")[0] != 0
    assert run(cli, "count --length 131072")[0] != 0
    assert run(cli, "count --length 8 --policy fancy")[0] != 0
    assert run(cli, "count --length 8 --ring fermat:1024")[0] == 0
    assert run(cli, "count --length 4096 --ring fermat:1024")[0] != 0  # above M = 2048


def test_rejects_malformed_ranges_and_rings(cli):  # cli_test.cpp:100-106, 123-133
    assert run(cli, "bench --min 16 --max 8")[0] != 0
    assert run(cli, "bench --min 0 --max 8")[0] != 0
    assert run(cli, "bench --min 1 --max 8589934592")[0] != 0
    assert run(cli, "bench --step-pct 0")[0] != 0
    assert run(cli, "bench --trials 0")[0] != 0
    assert run(cli, "verify --max-ell 6 --modulus 97 --two-adicity 5")[0] != 0
    assert run(cli, "verify --modulus 15 --max-ell 2")[0] != 0
    assert run(cli, "verify --modulus 17 --two-adicity 5 --max-ell 2")[0] != 0
    assert run(cli, "verify --max-ell 9")[0] != 0
    assert run(cli, "verify --ring fermat:100")[0] != 0
    assert run(cli, "verify --device cpu")[0] != 0
    assert run(cli, "")[0] != 0


@pytest.mark.gpu
def test_verify_passes_and_fault_fails(cli):  # cli_test.cpp:123-133; acceptance.cpp:207-245
    rc, out = run(cli, "verify --max-ell 4 --seed 1 --modulus 7681 --two-adicity 9")
    assert rc == 0, out
    assert "all 5 suites passed" in out
    rc, out = run(cli, "verify --max-ell 5")
    assert rc == 0, out
    for name in ("tft-oracle", "itft-inversion", "tft-bounds", "itft-bounds", "tft-smoothness"):
        assert name in out
    rc, out = run(cli, "verify --max-ell 4 --inject-fault")
    assert rc == 1, out
    assert "tft-oracle       FAIL" in out and "suites failed" in out


@pytest.mark.gpu
@pytest.mark.parametrize("ring", ["fermat:1024", "fermat:8192", "negacyclic:64,4611686018427387847"])
def test_verify_big_rings(cli, ring):
    rc, out = run(cli, f"verify --max-ell 4 --ring {ring}")
    assert rc == 0, out
    rc, out = run(cli, f"verify --max-ell 3 --inject-fault --ring {ring}")
    assert rc == 1, out


@pytest.mark.gpu
def test_bench_non_timing_columns_deterministic(cli):  # cli_test.cpp:79-98
    args = "bench --min 32 --max 128 --step-pct 25 --trials 1 --seed 9"
    ra, a = run(cli, args)
    rb, b = run(cli, args)
    assert ra == 0 and rb == 0
    la, lb = a.splitlines(), b.splitlines()
    assert len(la) == len(lb) > 2
    assert la[0] == "n,L,policy,wall_ns,butterflies"
    for x, y in zip(la[1:], lb[1:]):
        fx, fy = x.split(","), y.split(",")
        assert len(fx) == 5
        assert fx[:3] == fy[:3] and fx[4] == fy[4]
    rc, out = run(cli, "bench --min 100 --max 300 --step-pct 50 --trials 1 --ring fermat:8192")
    assert rc == 0 and out.splitlines()[0] == "n,L,policy,wall_ns,butterflies"


@pytest.mark.gpu
def test_compare_ratio_has_four_decimals(cli):  # cli_test.cpp:108-121
    rc, out = run(cli, "compare --min 16 --max 64 --step-pct 50 --trials 1")
    assert rc == 0
    lines = out.splitlines()
    assert lines[0] == "n,wall_ns_balanced,wall_ns_radix2,ratio"
    for line in lines[1:]:
        f = line.split(",")
        assert len(f) == 4 and len(f[3].split(".")[1]) == 4
