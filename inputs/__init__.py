"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NO concurrency-control arithmetic and NO transaction semantics.
It only produces inputs:

* the YCSB initial table S0 (``ycsb_rows``), SURVEY.md §8(c) reading Z11;
* the Zipf inverse-CDF threshold table that both batch generators search
  (``zipf_thresholds``), PAPER.md:457 ("following a Zipfian distribution"),
  SURVEY.md §8(c) reading Z13;
* the fixed key scramble multiplier (``scramble_mult``), reading Z13;
* tiny hand-shaped batches for brute-force tests (``random_batch``).

Both the device library (through its own CUDA copy of the row initialiser) and the
oracle receive exactly these arrays; nothing here is computed by either side.
"""
from .ycsb import (MASK64, mix64, ycsb_rows, ycsb_row, zipf_thresholds,
                   scramble_mult, random_batch, harmonic)  # noqa: F401
from . import tpcc  # noqa: F401
