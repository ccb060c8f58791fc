import sys; sys.path.insert(0,'.')
import paper_1204_0069_b200 as m
cfg = m.CONFIGS[0]
for arith in ("exact","fast"):
    with m.GpuContext(cfg.n, cfg.p, arith=arith) as ctx:
        b, X0, opts = m.make_problem_on_device(ctx, cfg)
        for i in range(3):
            t = ctx.solve(b, X0, opts)
            print(arith, t.iteration_count(), ctx.timing())
