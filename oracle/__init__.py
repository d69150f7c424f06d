"""ORACLE -- test infrastructure, not product code.

Plain, slow, obviously-correct CPU implementations of what the Nova hot path
computes (PAPER.md arXiv 2509.21301): the VLM forward (vlm.py), the partition
planner Eqs. 1-6 (planner.py), Algorithm 1 (scheduler.py) and the layer-wise
offload schedule Eqs. 7-8 (offload.py).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it.  It shares
no code with paper_2509_21301_b200/ and never imports it.

Parity pins: every function here is pinned by tests/test_oracle_*.py against
something other than itself (HF transformers in fp64, torch library routines,
paper-printed values, hand-derived worked examples, brute force, invariants).
No function is "parity unpinned".
"""
