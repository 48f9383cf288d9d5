"""CPU oracle for the B200 conv path -- test infrastructure only (see conv_oracle.py)."""
