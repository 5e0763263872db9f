"""CPU oracle (test infrastructure only; see msfv_oracle.py header)."""
