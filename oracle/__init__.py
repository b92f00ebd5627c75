"""TEST INFRASTRUCTURE: the CPU oracle (restatement of the reference
``gnncompose`` 0.1.0 hot path).  Imported only by tests/, the smoke check and
bench.py's CPU-baseline legs — never by the product package."""
