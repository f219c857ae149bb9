"""Per-rank device time of the four-step split, G ranks emulated on one GPU.

Checks the product, then times each rank's phases with CUDA events (columns_fwd, the
receive re-layout + rows, columns_inv; rank 0's gather re-layout + decode), so the
per-GPU compute of a G-GPU split can be read off a single B200.  --exchange alltoall: the
exchanges are not timed (local copies in the emulation; on a node they are NCCL all-to-alls
between the phases); --exchange peer (default): the phases store straight into the owning
ranks' buffers (here the other emulated ranks' buffers on the same GPU, on a node peer memory
over NVLink), so the exchange is inside the phase times and nothing runs between the phases
but a barrier.

  python tools/fourstep_phases.py --bits 24 --world 8 [--exchange peer|alltoall]
"""
import argparse
import json
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1503_04955_b200.fourstep import (_operands, _plan_and_limbs, _to_int, make_rank, run_virtual,  # noqa: E402
                                            run_virtual_peer)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=24)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--exchange", default="peer", choices=["peer", "alltoall"])
    args = ap.parse_args()
    N = 1 << args.bits
    r = random.Random(4)
    a = r.getrandbits(N) | 1 << (N - 1)
    b = r.getrandbits(N) | 1 << (N - 1)
    plan = _plan_and_limbs(a, b)
    dev = torch.device("cuda", 0)
    G = args.world
    ranks = [make_rank(plan, k, G, dev) for k in range(G)]
    A, B = _operands(plan, a, b, dev)

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    peer = args.exchange == "peer"
    if _to_int((run_virtual_peer if peer else run_virtual)(ranks, A, B)) != a * b:
        raise SystemExit("product mismatch")
    # timing: each phase enqueued `reps` times back to back (launch latency hidden, as in a
    # real run where the host runs ahead); every phase's device time is data independent
    if peer:
        z_peers = torch.tensor([fs.z.data_ptr() for fs in ranks], dtype=torch.int64, device=dev)
        x_peers = torch.tensor([fs.x.data_ptr() for fs in ranks], dtype=torch.int64, device=dev)
        g = ranks[0].gath.data_ptr()
        phases = {
            "columns_fwd": lambda fs: fs.phase_columns_peer(A, B, z_peers),
            "rows": lambda fs: fs.phase_rows_peer(x_peers),
            "columns_inv": lambda fs: fs.phase_finish_peer(g),
        }
    else:
        phases = {
            "columns_fwd": lambda fs: fs.phase_columns(A, B),
            "rows": lambda fs: fs.phase_rows(),
            "columns_inv": lambda fs: fs.phase_finish(),
        }
    res = {}
    for name, fn in phases.items():
        worst = 0.0
        for fs in ranks:
            fn(fs)
            torch.cuda.synchronize()
            e0 = ev()
            for _ in range(args.reps):
                fn(fs)
            e1 = ev()
            torch.cuda.synchronize()
            worst = max(worst, e0.elapsed_time(e1) / args.reps)
        res[name] = [worst]
    ranks[0].decode()
    torch.cuda.synchronize()
    e0 = ev()
    for _ in range(args.reps):
        ranks[0].decode()
    e1 = ev()
    torch.cuda.synchronize()
    res["decode"] = [e0.elapsed_time(e1) / args.reps]
    out = {k: round(sorted(v)[len(v) // 2], 4) for k, v in res.items()}
    out["compute_ms_per_rank"] = round(sum(out[k] for k in ("columns_fwd", "rows", "columns_inv")), 4)
    lay = ranks[0].stages.layout(G)
    out.update({"bits": args.bits, "world": G, "exchange": args.exchange,
                "exchange_bytes_per_rank_per_poly": 4 * lay["block_words"] * (G - 1) // G})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
