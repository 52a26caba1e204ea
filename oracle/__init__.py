"""CPU oracle for arXiv 2211.15716 (ImplicitGlobalGrid) -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct reference implementations written from
PAPER.md (and SPEC.md's readings where the paper is silent):

  heat3d  -- Fig. 1's heat solver on the whole global grid (C, fp64)
  grid    -- topology, global sizes, halo geometry, local<->global windows
  halo    -- update_halo! as dimension-sequential copies between numpy arrays

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  It shares no code with the CUDA
product (paper_2211_15716_b200/, include/) and neither imports the other.
"""
