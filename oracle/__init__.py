"""TEST INFRASTRUCTURE ONLY: CPU oracle for the POET-X hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product package (paper_2603_05500_b200) never imports
anything from here.
"""
