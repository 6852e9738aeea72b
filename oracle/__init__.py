"""G-VOM CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/gvom_oracle.c header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.  The product package never imports it.
"""
