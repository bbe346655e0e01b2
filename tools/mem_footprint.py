import sys; sys.path.insert(0,'.')
import torch
from paper_2505_13390_b200 import mgpbd, scenes
for name in ("block1.67M", "cloth2048"):
    torch.cuda.synchronize()
    f0,t=torch.cuda.mem_get_info()
    sc=scenes.make(name)
    ctx=mgpbd.Context.from_scene(sc, precision=1)
    ctx.step(sc.dt, 2)
    f1,_=torch.cuda.mem_get_info()
    print(name, sc.n_cons, "device bytes used %.2f GB" % ((f0-f1)/1e9), "bytes/constraint %.0f" % ((f0-f1)/sc.n_cons))
    ctx.close()
