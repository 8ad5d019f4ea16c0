"""CPU oracle package — test infrastructure only (see aol_oracle.py header)."""
