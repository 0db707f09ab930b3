"""Plain CPU oracle of the LoPA verify step (TEST INFRASTRUCTURE ONLY; see lopa_oracle.py)."""
