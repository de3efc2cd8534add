"""One rank of a multi-process run of the P > 1 path (launched by tests/test_gpu_multiproc.py through torchrun): real
processes, CUDA IPC mappings of every peer's entity shard and exchange block (kge_export / kge_connect), cross-process
system-scope device barriers. With fewer GPUs than ranks every rank shares cuda:0 (the IPC and barrier protocol is the
same; the contexts time-slice). Rank 0 checks the result against the oracle's P-rank union step (reading c.13)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2004_08532_b200 import kge  # noqa: E402


def main():
    model, steps, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    lag = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    extra = sys.argv[5] if len(sys.argv) > 5 else ""  # "repartition" | "placement" | ""
    opts = {"repartition": dict(repartition=1), "placement": dict(placement=1, neg_local=1)}.get(extra, {})
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = rank if torch.cuda.device_count() >= ws else 0
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    gr = synth.graph("tiny")
    trip = gr.triples()
    B, g, k, d = 128, 32, 32, 32
    cfg = kge.Config(model=model, n_entities=gr.n_entities, n_relations=gr.n_relations, dim=d, batch_size=B,
                     chunk_size=g, neg_k=k, neg_precision="fp32", world_size=ws, rank=rank, lag=lag, **opts)
    h = kge.init_distributed(cfg, *trip)
    h.set_option("barrier_ms", 120000)
    losses = h.train_step(steps)
    h.flush()
    own = np.arange(rank, gr.n_entities, ws)
    rows = h.get_rows(0, own)
    st = h.get_rows(3, own)
    rids = np.arange(gr.n_relations)
    owner = np.array([h.relation_owner(r) for r in rids])
    mine = rids[(owner == rank) | ((owner == -1) & (rank == 0))]
    rel = h.get_rows(1, mine)
    res = [None] * ws
    dist.all_gather_object(res, dict(losses=losses, own=own, rows=rows, st=st, rids=mine, rel=rel))
    if rank == 0:
        import oracle as O  # test infrastructure: the check runs in the test's worker, never in the product
        orc = O.Trainer(model, gr.n_entities, gr.n_relations, d, B, g, k, world_size=ws, triples=trip, lag=lag, **opts)
        lo = orc.train(steps)
        orc.flush()
        lg = sum(r["losses"].astype(np.float64) for r in res)
        E = np.zeros((gr.n_entities, d))
        S = np.zeros(gr.n_entities)
        for r in res:
            E[r["own"]] = r["rows"]
            S[r["own"]] = r["st"][:, 0]
        R = np.zeros((gr.n_relations, cfg.dim if model != "rotate" else d // 2))
        for r in res:
            R[r["rids"]] = r["rel"]
        ids = np.arange(gr.n_entities)
        report = {"loss_rel": float(np.max(np.abs(lg - lo) / np.abs(lo))),
                  "rows": float(np.abs(E - orc.get_rows(0, ids)).max()),
                  "states": float(np.abs(S - orc.get_rows(3, ids)[:, 0]).max()),
                  "rel": float(np.abs(R - orc.get_rows(1, rids)).max()),
                  "steps": steps, "world_size": ws, "device_count": torch.cuda.device_count()}
        with open(out, "w") as f:
            json.dump(report, f)
    dist.barrier()
    h.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
