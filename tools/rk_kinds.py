"""C3 re-check cases and kernel times per max-family measure (Linf, W1inf, W1infsum alone, then together)."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import cilgen, bench
import paper_2203_14742_b200 as cil
from paper_2203_14742_b200 import _capi
dev=torch.device("cuda"); grid=(2,128,128); N=2000; M=20
A=cilgen.make_set(cilgen.config_seed(3),0,N,grid,device=dev); B=cilgen.make_set(cilgen.config_seed(3),1,N,grid,device=dev)
Rall=torch.tensor(bench.pilot_radii_all(A,B,grid,M,0x3F),dtype=torch.float64,device=dev)
for name,mask,rows in (("Linf",0x02,[1]),("W1inf",0x10,[4]),("W1infsum",0x20,[5]),("maxfam",0x32,[1,4,5])):
    R=Rall[rows]; ws=cil.Workspace()
    for _ in range(2): cil.features(A,B,grid,mask,R,ws=ws)
    torch.cuda.synchronize(); _capi.prof_enable(True)
    for _ in range(3): cil.features(A,B,grid,mask,R,ws=ws)
    torch.cuda.synchronize(); _capi.prof_enable(False); p=_capi.prof_read()
    n,_=cil.recheck_count(1,N,N,grid,mask,M,cil.ENGINE_AUTO,ws=ws)
    print(name, "cases", n, {k:round(v[0]/3,3) for k,v in p.items() if v[1]})
