import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1508_04458_b200 as W
from paper_1508_04458_b200 import configs
from oracle import oracle as O
from wam_testutil import problem_inputs
name = sys.argv[1] if len(sys.argv) > 1 else "tiny3d"
cfg, p, _, I0, d = problem_inputs(name, O, W)
c = W.Context(0)
c.set_geometry(configs.geometry(cfg, W.Geometry))
c.set_haar_dim(3)
c.set_data(d, I0)
c.wam_init(cfg["L"])
r = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
print("ok", r[-1])
