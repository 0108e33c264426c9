import sys, os
sys.path.insert(0, os.getcwd())
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller
w = workload.make("c0")
c = Controller(w.params, w.bounds, w.sg, w.cost, precision="fp32", noise="philox")
c.set_mlp(w.mlp); c.set_costmap(w.costmap)
for _ in range(3):
    c.mpc_step(w.x0[0])
print("ok")
