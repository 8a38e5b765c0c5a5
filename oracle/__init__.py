"""DF11 CPU oracle (TEST INFRASTRUCTURE ONLY).

A plain, slow, obviously-correct CPU implementation of what the DF11 hot path computes, written from
the paper (arXiv 2504.11651, PAPER.md) step by step.  Only tests/, __graft_entry__.smoke() and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import, call, link or execute anything in
this directory.  The product package ``paper_2504_11651_b200`` never imports it and shares no code
with it (no kernels, headers, helpers, tables or constant generators).

Pins: every function here is checked by tests/test_oracle_*.py against the paper's worked examples
(tests/golden/), brute force on tiny inputs, closed forms and invariants.  Parity status per function
is listed in DESIGN.md §4.
"""
from .oracle import (FormatError, VALUE_FORMATS, WORD_DTYPE, build_oracle, compose,  # noqa: F401
                     compose_v, compressed_bytes, decode_alg1, decode_alg1_blocks, decode_alg1_range,
                     decode_sequential, decode_sequential_blocks, encode, entropy_bits, histogram, residual_array_bytes, residual_bits,
                     split, split_v, vf_code)
from . import huffman  # noqa: F401
