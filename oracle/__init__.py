"""CPU oracles for the FlexDeMo optimizer step -- TEST INFRASTRUCTURE ONLY (see oracle.py)."""
