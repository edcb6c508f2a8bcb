"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 CPU implementation of the P-ERK multirate DGSEM step written
from the paper and the readings of SURVEY.md §8(c).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
`bench.py --impl reference`) may import, call or execute anything here; the
product path (paper_2403_05144_b200) never does.  Shares no code with the CUDA
path.  Parity-unpinned functions: none implemented that are unpinned (the BR1
Navier-Stokes operator is not implemented yet).
"""
