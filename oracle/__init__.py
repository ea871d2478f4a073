"""TEST INFRASTRUCTURE ONLY (see oracle/oracle.py). Not part of the product."""
