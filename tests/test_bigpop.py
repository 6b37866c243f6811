"""-m "not gpu": the shared-memory parallel population (tests/bigpop.py, used by the
configs[4]-size parity tests) is byte-identical to inputs.tpcc.population."""
import numpy as np

from inputs import tpcc as IT


def test_parallel_population_matches_serial():
    import bigpop
    P = bigpop.population(5, 10, procs=4, chunk=3)
    try:
        S = IT.population(5, 10)
        for k in S:
            assert np.array_equal(P[k], S[k]), k
    finally:
        P.close()
