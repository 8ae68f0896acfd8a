"""TEST INFRASTRUCTURE ONLY: CPU oracle for the Shor hot path (see oracle.py)."""
