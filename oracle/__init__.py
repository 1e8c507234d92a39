"""CPU oracle package (test infrastructure only; see ``port.py``)."""
