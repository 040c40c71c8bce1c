"""TEST INFRASTRUCTURE ONLY: CPU checkers for the VLBM hot path (see oracle.py).
Never imported by the product package."""
