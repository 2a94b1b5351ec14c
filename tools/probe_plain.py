import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, json
import paper_2211_03339_b200 as mpj, workloads as W
n=1024
for kind,gen,mode in (("uniform",W.example1,4),("clustered",W.example2,4)):
    A,lam=gen(n,1e3,mode,W.seed_for(2,mode,1e3))
    At=torch.from_numpy(A).cuda()
    for plain in (False,True):
        r=mpj.eig(At,plain=plain); torch.cuda.synchronize()
        mpj.profile_reset(); mpj.profile_enable(True)
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); r=mpj.eig(At,plain=plain); e1.record(); torch.cuda.synchronize()
        mpj.profile_enable(False)
        ks={k: [round(x,5) for x in mpj.profile_get(k)] for k in ("block_apply_f64","block_solve_f64","block_apply_f32","block_solve_f32")}
        print(kind, "plain" if plain else "mp", round(e0.elapsed_time(e1),2), "ms sweeps", r.sweeps, r.report.t_jacobi, ks, "rot", r.report.rotations)
