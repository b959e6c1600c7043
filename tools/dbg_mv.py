import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
sys.path.insert(0, "/root/repo/tests"); from conftest import golden
from paper_2007_04560_b200.grid import Grid, BoundaryCondition
from paper_2007_04560_b200.physics import Params, State
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian
for tag in ["3d_neu","3d_per","3d_neu_big"]:
    z=golden(f"stencil_{tag}.npz")
    counts=tuple(int(c) for c in z["counts"]); bc=BoundaryCondition.PERIODIC if bool(z["periodic"]) else BoundaryCondition.NEUMANN
    g=Grid(counts,(1.0,)*3,bc); P=Params(4.0,2.0,0.005,0.1,0.001)
    st=lambda u,v: State.from_interior(g,u,v,device="cuda:0")
    prob=StepProblem.create(g,P,st(z["uo"],z["vo"]),float(z["dt"]))
    J=assemble_jacobian(prob,st(z["un"],z["vn"]))
    y=J.matvec(torch.tensor(z["w"],device="cuda:0")).cpu().numpy()
    d=np.abs(y-z["Jw"]).reshape(counts[2],counts[1],counts[0],2)
    print(tag, counts, "max err per z plane (u, v):")
    for k in range(counts[2]): print("  ",k, d[k,:,:,0].max(), d[k,:,:,1].max())
