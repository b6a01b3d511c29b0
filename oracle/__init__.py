"""SMART fp64 oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl
reference`` legs may import this package.  The product path
(paper_2604_09731_b200) never imports it and shares no code with it.
"""
