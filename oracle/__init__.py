"""CPU oracle (test infrastructure only — see mds_oracle.py header)."""
