"""CPU oracle (test infrastructure only; see pipeline_oracle.py header)."""
