"""CPU oracle package - TEST INFRASTRUCTURE ONLY (see oracle/ppa_oracle.cpp header)."""
