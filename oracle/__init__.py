"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see gvo_oracle.py)."""
