"""One on-device random_spd generation (the reference's make_problem matrix) of
size n = argv[1], for ncu launch lists of the refgen kernels:
    ncu --metrics gpu__time_duration.sum -s 4000 -c 4 python tools/rg_one.py 4096
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1204_0069_b200 as m  # noqa: E402

n = int(sys.argv[1])
with m.GpuContext(n, 2) as ctx:
    ctx.gen_A("random_spd", 7, 0, 1e3)
