"""Synthetic workload generator of the BASELINE configs (bench, tests, checker inputs)."""
