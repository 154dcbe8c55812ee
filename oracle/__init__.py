"""CPU oracle for the SwiftSpec tree-verify step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product (paper_2506_11309_b200)
never imports, links or executes it, and this package never imports the
product: the two share no code except the input generators in synth/.
"""
from .swiftspec_oracle import *  # noqa: F401,F403
