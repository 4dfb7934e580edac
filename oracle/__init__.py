"""fp64 CPU oracle of the 3DGUT forward rasterizer — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product package
(paper_2412_12507_b200/) never imports it and the product .so never links it.
"""
