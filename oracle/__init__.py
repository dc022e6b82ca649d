"""CPU checkers (test infrastructure only; see oracle/bind.py)."""
