"""oracle/ — TEST INFRASTRUCTURE ONLY (see cqs_oracle.py header).  Importable only from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs."""
