"""CPU oracles for parity testing (test infrastructure only; see pyoracle.py)."""
