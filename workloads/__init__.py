"""Synthetic workloads: seeded input generator (gen.py) and config graph specs (configs.py).

Shared by the oracle and the CUDA-path harness; contains no method arithmetic.
"""
