"""CPU oracle (test infrastructure only; see oracle/hmbem_oracle.cpp)."""
