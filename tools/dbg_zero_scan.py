import sys, torch
sys.path.insert(0, '/root/repo')
from paper_1207_1746_b200 import gscl
gscl.init(0,1,device=0)
for op, N, h_c in [("JACOBI7", 512, None), ("VARCOEF8", 768, 0), ("VARCOEF8", 384, 0)]:
    u = gscl.Grid(N,N,N,1).fill_random(12071746, 0)
    ins=[u]
    if op == "VARCOEF8":
        ins += [gscl.Grid(N,N,N,0).fill_random(12071746, 2+i, 0.125) for i in range(7)]
    out = gscl.Grid(N,N,N,1)
    gscl.do_all(op, ins, out); gscl.sync()
    v = out.device_view(); ox = out.origin_offset % out.pitch
    I = v[1:1+N, 1:1+N, ox:ox+N]
    z = (I == 0)
    nz = int(z.sum())
    print(op, N, "zeros:", nz, flush=True)
    if nz:
        idx = z.nonzero()
        print(" first", idx[0].tolist(), "last", idx[-1].tolist(), "zmin", int(idx[:,0].min()), "ymin", int(idx[:,1].min()), "xmin", int(idx[:,2].min()))
        zz = z.any(dim=2).any(dim=1).nonzero().flatten().tolist()
        print(" planes with zeros:", zz[:5], '...', zz[-5:], len(zz))
    for g in ins+[out]: g.destroy()
    torch.cuda.empty_cache()
