"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see packkv_oracle.py header)."""
