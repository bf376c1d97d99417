"""DASH deterministic attention backward for B200 (sm_100a) -- Python binding of libdash.so."""
