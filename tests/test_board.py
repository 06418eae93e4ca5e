"""The balancer's cross-rank agreement board (csrc/board.h — what multi-rank
worlds use to max-reduce per-path times at every decision point) across real
processes on the CPU: 2/3/4/8 forked ranks, 400 decision points each with 1-150
values and random pauses, every rank sees the elementwise max; a rank that stops
publishing makes the others time out (flxInternalError in the library) rather
than hang."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def board_test(tmp_path_factory):
    exe = tmp_path_factory.mktemp("board") / "board_test"
    subprocess.run(["g++", "-O2", "-std=c++17", "-Wall", "-Werror",
                    f"-I{ROOT / 'paper_2510_15882_b200' / 'csrc'}",
                    str(ROOT / "tools" / "board_test.cpp"), "-o", str(exe)], check=True)
    return exe


@pytest.mark.parametrize("ranks", [2, 3, 4, 8])
def test_board_agreement_across_processes(board_test, ranks):
    out = subprocess.run([str(board_test), str(ranks), "400"], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stdout)
