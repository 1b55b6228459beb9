"""Plain fp64 CPU oracle (test infrastructure only; see oracle/cwb_oracle.h)."""
