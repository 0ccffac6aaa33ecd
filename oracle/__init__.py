"""CPU oracle for the HB-CSF path — TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
legs.  The product package (paper_1904_03329_b200) never imports it.
"""
