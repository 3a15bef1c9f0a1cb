import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2007_11919_b200 as mds
from paper_2007_11919_b200.synthetic import scenario
x = scenario(3000, 10, 5, seed=17)
x[1234, 3] = np.inf
for name, prm in [("divide", dict(r=5, l=400, c=10, seed=7)), ("interpolate", dict(r=5, l=1000, seed=7)),
                  ("fast", dict(r=5, l=400, s=10, seed=7))]:
    try:
        mds.run_algorithm(name, x, mds.AlgorithmParams(**prm))
        print(name, "no error!")
    except mds.InvalidInputError as e:
        print(name, "ok", e)
