"""Worker for tests/test_multirank.py (one process per rank, gloo rendezvous on 127.0.0.1).

mode "exchange": exercises the gloo exchange callbacks through ctypes function pointers (CPU only).
mode "fit": 2 ranks share cuda:0 through the host exchange; SYN-v1 rows sharded by rank.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch.distributed as dist


def main():
    mode, out = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2506_02007_b200.dist import gloo_exchange
    ag, ar = gloo_exchange()
    if mode == "exchange":
        from paper_2506_02007_b200 import ALLGATHER_FN, ALLREDUCE_FN
        fag, far = ALLGATHER_FN(ag), ALLREDUCE_FN(ar)
        send = np.arange(5, dtype=np.float64) + 10 * rank
        recv = np.empty(5 * world)
        assert fag(None, send.ctypes.data, recv.ctypes.data, 40) == 0
        res = {"gather": recv}
        for dt, code in ((np.float64, 0), (np.int64, 1)):
            for op in (0, 1, 2):
                b = (np.array([3, -1, 7], dtype=dt) * (rank + 1))
                assert far(None, b.ctypes.data, 3, code, op) == 0
                res[f"r{code}{op}"] = b
        np.savez(out + f".{rank}.npz", **res)
    else:
        import paper_2506_02007_b200 as es
        n = int(sys.argv[3])
        ctx = es.Context(0, rank, world, exchange=(ag, ar))
        ds = es.Dataset.generate(42, n, 16, 8, ctx=ctx)
        m = es.fit_em(ds, 8, init="random", tol=0.0, max_iter=8, seed=7)
        d, ld = es.calibrate_threshold(m, ds, 0.01, n_train=n // 2, return_log=True)
        r = es.detect(m, ds, log_delta=ld)
        mk = es.fit_em(ds, 4, init="kmeans++", tol=0.0, max_iter=3, seed=5)
        kb = es.kmeans_baseline(ds, 4, q=0.02, seed=3)
        pr = es.run_pipeline(ds, 4, quantile_q=0.02, seed=1, max_iter=10)
        np.savez(out + f".{rank}.npz", w=m.weights, mu=m.means, cov=m.covariances,
                 per=m.fit_report.per_iteration_log_likelihoods, final=m.fit_report.final_log_likelihood,
                 delta=d, ld=ld, idx=r.anomaly_indices, nflag=r.n_flagged, off=ds.row_offset,
                 kmu=mk.means, kw=mk.weights, kbc=kb.centroids, kbt=kb.threshold, kbn=kb.n_flagged,
                 kbf=kb.flags, kbi=kb.iterations, pmu=pr.model.means, pmean=pr.mean, pscale=pr.scale,
                 pdelta=pr.report.delta, pn=pr.report.n_flagged, pf=pr.report.flags)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
