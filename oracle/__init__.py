"""CPU oracle package — test infrastructure only (see fmm_oracle.py header)."""
