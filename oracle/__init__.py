"""CPU oracle of the LRBMS online step -- test infrastructure only (see lrbms_oracle.py header)."""
