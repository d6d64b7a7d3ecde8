"""CPU oracle for the MoE-layer hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import or execute anything under oracle/. The
product path (paper_2305_13525_b200/) never imports it and has no CPU
fallback. The oracle shares no code with the CUDA path.
"""
from .moe_oracle import *  # noqa: F401,F403
