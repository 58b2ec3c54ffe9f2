"""Benchmark / evidence scripts and the synthetic-input generator (not the product)."""
