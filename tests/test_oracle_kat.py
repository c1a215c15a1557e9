"""The numpy oracle against the reference's own known-answer tests (CPU)."""
import numpy as np
import pytest

from tests import kat
from tests.impls import OracleImpl

IMPL = OracleImpl()


@pytest.mark.parametrize("check", kat.PROPAGATOR_KATS + kat.TRANSFER_KATS + kat.ENERGY_KATS + kat.PROCRUSTES_KATS, ids=lambda f: f.__name__)
def test_oracle_known_answers(check):
    check(IMPL)


def test_oracle_repeated_step_bitwise():
    manual, out, out2 = kat.repeated_step_bitwise(IMPL)
    assert np.array_equal(manual[0], out[0]) and np.array_equal(manual[1], out[1])
    assert np.array_equal(out[0], out2[0]) and np.array_equal(out[1], out2[1])
