import sys; sys.path.insert(0,'/root/repo')
import paper_2203_13382_b200 as P
for kw in (dict(n_x=1024, n_t=512, dim=2, wave_speed="B4", p=5, schedule=8, seed=4, u0="sin4"),
           dict(n_x=512, n_t=256, dim=2, wave_speed="B4", p=3, schedule=4, seed=3, u0="sin4")):
    lv = P.build_hierarchy(P.SolverConfig(**kw))
    print(kw["n_x"], [(l.n_steps, l.kind, l.separable) for l in lv])
