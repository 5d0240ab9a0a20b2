"""Small 1D + 2D solves (all phase kinds, every cluster size, the two-CTAs-per-SM
phase) for memory-checker runs where a checker is available."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_13382_b200 as P  # noqa: E402

for kw in (dict(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4),
           dict(n_x=4096, n_t=64, wave_speed="B2", p=3, schedule=4),
           dict(n_x=64, n_t=64, wave_speed="C2", p=1, schedule=4, relaxation="F"),
           dict(n_x=64, n_t=128, wave_speed="C1", p=1, schedule=8, max_levels=2),
           dict(n_x=16, n_t=64, dim=2, wave_speed="C5", p=3, schedule=4),
           dict(n_x=32, n_t=64, dim=2, wave_speed="B4", p=5, schedule=4, operator_kind="forward_euler",
                max_levels=2)):
    cfg = P.SolverConfig(**kw, max_iters=3)
    rep, U = P.solve(cfg)
    print(kw, rep.iterations, rep.status)

# every cluster size on the corrected 1D phases / sweeps (n = 4096: CS 2..16;
# n = 16384: the global-gather form), and the two-CTAs-per-SM phase (level 1
# of n_t = 2400, m = 4: 150 row chains > one CTA per SM)
for pol, kw in (("cluster2", dict(n_x=4096, n_t=64, wave_speed="B2", p=3, schedule=4)),
                ("cluster4", dict(n_x=4096, n_t=64, wave_speed="B2", p=5, schedule=4)),
                ("cluster8", dict(n_x=1024, n_t=128, wave_speed="C3", p=3, schedule=4, max_levels=2)),
                ("cluster16", dict(n_x=16384, n_t=64, wave_speed="B2", p=5, schedule=8)),
                ("auto", dict(n_x=4096, n_t=2400, wave_speed="B2", p=3, schedule=4, max_levels=3))):
    prev = P.set_launch_policy(pol)
    cfg = P.SolverConfig(**kw, max_iters=1)
    rep, U = P.solve(cfg)
    P.set_launch_policy(prev)
    print(pol, kw, rep.iterations, rep.status)
print("ok")
