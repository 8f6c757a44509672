import sys, os, torch
sys.path.insert(0, os.getcwd())
import cilgen, bench
import paper_2203_14742_b200 as cil
dev=torch.device("cuda"); grid=(2,128,128); N=2000; M=20
A=cilgen.make_set(cilgen.config_seed(3),0,N,grid,device=dev); B=cilgen.make_set(cilgen.config_seed(3),1,N,grid,device=dev)
Rall=torch.tensor(bench.pilot_radii_all(A,B,grid,M,0x3F),dtype=torch.float64,device=dev)
R=Rall[[1,4,5]]; ws=cil.Workspace()
for _ in range(2): cil.features(A,B,grid,0x32,R,ws=ws)
torch.cuda.synchronize()
