import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2506_02007_b200 as es
ctx = es.Context(0)
m1 = es.GmmModel(np.array([1.0]), np.array([[0.0]]), np.array([[[1.0]]]))
for name, f in [("cld", lambda: es.component_log_density(m1, [0.0], 0, ctx=ctx)),
                ("gen", lambda: es.Dataset.generate(42, 4096, 8, 4, ctx=ctx)),
                ("fit", lambda: es.fit_em(es.Dataset.generate(42, 4096, 8, 4, ctx=ctx), 4, init="random", max_iter=3))]:
    try:
        print(name, f())
    except Exception as e:
        print(name, "FAILED", e)
