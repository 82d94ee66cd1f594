"""Two (or more) processes, one slab each, stepping through the CUDA-IPC halo
push (imb_team_connect_ipc). Every rank uses the same GPU here, so this checks
the protocol and the cross-process mapping, not NVLink bandwidth. Rank 0
compares the gathered slabs with a single-slab run bit for bit and exits 0
on success. Launched by tests/test_gpu_parity.py under a timeout:

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29533 tests/mp/ipc_ring.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1507_01265_b200 import mpdata  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, m, l = 12 * world + 5, 20, 64
    iord, nonos, fp64 = (int(v) for v in (sys.argv[1:4] if len(sys.argv) >= 4 else (2, 1, 1)))
    opts = mpdata.Options(iord, bool(nonos), bool(fp64))
    shares = [n // world + (1 if r < n % world else 0) for r in range(world)]
    i0 = sum(shares[:rank])
    team = mpdata.Team(n, m, l, opts, device=0, i0=i0, ni=shares[rank])
    upload = os.environ.get("IPC_RING_UPLOAD") == "1"
    fields = None
    if upload:
        # host-uploaded x, u, v, w, h (uniform-random, divergent Courant
        # numbers): the static halos must then come from the neighbours
        from oracle import oracle as O
        fields = O.init_fields(0, n, m, l, seed=13, dtype=opts.dtype)
        team.upload_all(*(f[i0:i0 + shares[rank]] for f in fields))
    else:
        team.init_recipe(2, 11)
    blobs = [None] * world
    dist.all_gather_object(blobs, team.ipc_export())
    team.connect_ipc(blobs[(rank - 1) % world], blobs[(rank + 1) % world], world, rank)
    dist.barrier()
    extra = int(os.environ.get("IPC_RING_STEPS", "0"))  # stress runs: more steps per call
    team.run(3 + extra)
    team.run(2)  # continues across calls
    # host-buffer step through the same ring (rewrite epochs)
    x = team.download("x")
    out = np.empty_like(x)
    team.step_host(x, out)
    parts = [None] * world
    dist.all_gather_object(parts, out)
    ok = True
    if rank == 0:
        with mpdata.Team(n, m, l, opts, device=0) as t:
            if upload:
                t.upload_all(*fields)
            else:
                t.init_recipe(2, 11)
            t.run(6 + extra)
            want = t.download("x")
        got = np.concatenate(parts, axis=0)
        ok = bool(np.array_equal(got, want))
        print(f"ipc ring world={world} iord={iord} nonos={nonos} fp64={fp64} upload={upload}: "
              f"{'bit-identical' if ok else 'MISMATCH'}", flush=True)
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    dist.barrier()
    team.close()
    dist.destroy_process_group()
    sys.exit(0 if flag[0] else 1)


if __name__ == "__main__":
    main()
