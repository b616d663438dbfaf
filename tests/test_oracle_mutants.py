"""Test-of-tests: each deliberately broken oracle build (oracle.c ORACLE_MUTANT=k,
one plausible mistake each: dropped term, wrong sign, swapped branch, wrong
estimator, ignored layout ...) must trip at least one pin."""
import pytest

import oracle
from tests.oracle_pins import PINS

MUTANTS = list(range(1, 15))


@pytest.mark.parametrize("mutant", MUTANTS)
def test_mutant_is_caught(mutant):
    o = oracle.load(mutant)
    assert o.mutant == mutant
    caught = []
    for pin in PINS:
        try:
            pin(o)
        except AssertionError:
            caught.append(pin.__name__)
    assert caught, f"mutant {mutant} passed every pin"
