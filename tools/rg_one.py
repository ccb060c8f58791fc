import sys; sys.path.insert(0, '/root/repo')
import paper_1204_0069_b200 as m
n = int(sys.argv[1])
with m.GpuContext(n, 2) as ctx:
    ctx.gen_A("random_spd", 7, 0, 1e3)
