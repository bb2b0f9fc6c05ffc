"""CPU oracle (test infrastructure only; see pf_oracle.py header)."""
