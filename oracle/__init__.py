"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import, call, link or execute anything under
oracle/.  The product path (paper_2409_05205_b200/) never imports it and
shares no code with it.  See oracle/ref.py for the definitions, their
citations and the list of pins; "parity unpinned" items are listed in
DESIGN.md.
"""
