"""CPU: the period-window parity machinery of tests/test_full_size.py, run with the C
restatement (oracle/gn_oracle.c) as the "full problem" in place of the GPU, against the
compiled reference's window problems -- so the window maps, the edge-column rule and the
bit-exact KKT comparison are themselves checked before they judge the GPU path."""
import pytest

from oracle import bindings as B
from paper_2405_14032_b200.network import synthetic_case
from test_full_size import build_full, check_window_callbacks, check_window_kkt

T = 12
WINDOWS = [(0, T), (0, 3), (4, 3), (9, 3), (5, 2)]


@pytest.fixture(scope="module")
def oracle_full():
    if not B.ref_available():
        pytest.skip("oracle/_ref not built")
    raw = synthetic_case(160, 260, 30, 120, seed=21, parallel_lines=4, shared_gens=3)
    return build_full("synthetic160", raw, T, backend="oracle")


@pytest.mark.parametrize("win", WINDOWS, ids=[f"T0={a}-TW={b}" for a, b in WINDOWS])
def test_window_machinery_on_oracle(oracle_full, win):
    check_window_callbacks(oracle_full, *win)
    check_window_kkt(oracle_full, *win)
