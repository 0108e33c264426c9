import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02342_b200 import workload
from paper_1707_02342_b200.api import Controller
C, K = int(sys.argv[1]), int(sys.argv[2])
w = workload.make("c3", samples=K, controllers=C)
c = Controller(w.params, w.bounds, w.sg, w.cost, hidden=32, precision="fp32", noise="philox", n_controllers=C)
c.set_mlp(w.mlp); c.set_costmap(w.costmap)
x = w.x0 if C > 1 else w.x0[0]
c.closed_loop(x, 3, traces=False)
