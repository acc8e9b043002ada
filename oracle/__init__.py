"""CPU oracle of the FreqCache decision path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg; the product package never imports it.
"""
