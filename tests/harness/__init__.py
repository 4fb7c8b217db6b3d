"""Measurement harnesses that call the oracle (test infrastructure): full-size
parity and certificates (run_configs.py), the paper's accuracy tables
(accuracy_table.py), oracle timings at the tuned ω (oracle_sor_time.py).
They live under tests/ because only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may touch oracle/."""
