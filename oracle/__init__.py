"""CPU oracle for arXiv 2005.10494 (TEST INFRASTRUCTURE ONLY — see oracle.py header)."""
