"""TPC-C input generators (filled in with the TPC-C rows of SURVEY.md §8)."""
