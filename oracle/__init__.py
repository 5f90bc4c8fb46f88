"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path (see oracle.py)."""
