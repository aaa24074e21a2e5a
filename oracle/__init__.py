"""CPU oracle for the BHPP query path -- test infrastructure only (see cpu_oracle.py)."""
