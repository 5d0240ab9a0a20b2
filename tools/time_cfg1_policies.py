import time, torch, sys
sys.path.insert(0, '.')
import bench
import paper_2203_13382_b200 as P
for pol in ["cta", "cluster", "cta", "cluster"]:
    P.set_launch_policy(pol)
    cfg = P.SolverConfig(**bench.CONFIGS["cfg1"])
    lv = P.build_hierarchy(cfg)
    for w in range(3):
        P.solve(cfg, lv, output="device")
    torch.cuda.synchronize()
    ts = []
    for r in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); rep, _ = P.solve(cfg, lv, output="device"); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(pol, rep.iterations, min(ts), sorted(ts)[5])
