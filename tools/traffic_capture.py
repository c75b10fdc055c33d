"""DRAM traffic of the attention kernel for bench.py's roofline.traffic.

Runs the attention launches of ONE step of the rank bench.py reports (the
busiest rank of the workload of N GPUs: config 2 at N=1, config 3 at N>1) on
one GPU — ring rounds against KV buffers of the right size — so that ncu can
measure them; then, with --collect, turns the ncu CSV into
profiles/r02_attn_traffic.json keyed by N.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
      -k regex:attn_fwd_kernel --csv --log-file gpurun_out/traffic_nN.csv \\
      python tools/traffic_capture.py N
  python tools/traffic_capture.py --collect N gpurun_out/traffic_nN.csv
"""
import csv
import json
import os
import sys

sys.path.insert(0, ".")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r02_attn_traffic.json")


def busiest_program(n):
    from paper_2509_21841_b200 import plan as P, remap as M, schedule as S, workloads as W
    from paper_2509_21841_b200.program import build_rank_program
    batch = W.c2_batch("github", 0) if n == 1 else W.c3_batch(n)
    cluster = W.cluster_for(batch, n)
    plan = P.build_plan(batch, cluster)
    sched = S.build_schedule(plan)
    res = M.solve_remap(plan.tokens_per_rank, M.cost_matrix(cluster))
    progs = [build_rank_program(plan, sched, r, 32, res) for r in range(n)]
    return max(progs, key=lambda p: p.pairs_per_head())


def algorithmic_bytes(prog):
    """Bytes each launch must move once: local — q, k, v read, o (bf16) and
    lse written; ring round r — its query rows and the held KV set read, the
    fp32 running state (O, m, l) read unless r is the first round and written
    unless it is the last, o + lse written by the last round."""
    local_rows = sum(f.length for f in prog.local_frags)
    total = local_rows * (32 + 16) * 128 * 2 + local_rows * 32 * (128 * 2 + 4)
    for rp in prog.rings:
        g = rp.group_size
        for r, rr in enumerate(rp.rounds):
            qrows = sum(f.length for f in rr.frags)
            state = qrows * 32 * (128 + 2) * 4
            total += qrows * 32 * 128 * 2 + rr.kv_rows * 16 * 128 * 2
            total += (state if r > 0 else 0) + (state if r < g - 1 else 0)
            if r == g - 1:
                total += qrows * 32 * (128 * 2 + 4)
    return total


def run(n):
    import torch

    from paper_2509_21841_b200 import ops
    from paper_2509_21841_b200.engine import DeviceProgram
    prog = busiest_program(n)
    dev = torch.device("cuda", 0)
    dp = DeviceProgram(prog, dev)
    t = prog.rows
    q = torch.randn(t, 32, 128, device=dev, dtype=torch.bfloat16)
    k = torch.randn(t, 8, 128, device=dev, dtype=torch.bfloat16)
    v = torch.randn(t, 8, 128, device=dev, dtype=torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(32, max(t, 1), device=dev)
    if dp.local.n:
        ops.attn_fwd(q, k, v, dp.local.items, dp.local.n, dp.local.segs, o, lse)
    for rp, (pack, rounds) in zip(prog.rings, dp.rings):
        buf = torch.randn(max(rp.held_rows), 2, 8, 128, device=dev).to(torch.bfloat16)
        st_o = torch.zeros(max(rp.state_rows, 1), 32, 128, device=dev)
        st_ml = torch.zeros(2, 32, max(rp.state_rows, 1), device=dev)
        for r, work in enumerate(rounds):
            if work.n:
                nk = rp.rounds[r].kv_rows
                ops.attn_fwd(q, buf[:nk, 0], buf[:nk, 1], work.items, work.n, work.segs, o, lse, st_o, st_ml)
    torch.cuda.synchronize()
    print("rank", prog.rank, "pairs/head", prog.pairs_per_head(), "launches",
          int(dp.local.n > 0) + sum(w.n > 0 for _, rs in dp.rings for w in rs))


def collect(n, path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rd = csv.DictReader(lines)
    per = {}
    for r in rd:
        if "attn_fwd_kernel" not in r.get("Kernel Name", ""):
            continue
        per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    for lid in sorted(per, key=int):
        m = per[lid]
        rows.append({"read": m.get("dram__bytes_read.sum", 0.0), "write": m.get("dram__bytes_write.sum", 0.0),
                     "ns": m.get("gpu__time_duration.sum", 0.0)})
    prog = busiest_program(n)
    doc = json.load(open(OUT)) if os.path.exists(OUT) else {}
    doc[f"n{n}"] = {
        "workload": "C2 github seed 0 (all local)" if n == 1 else f"C3 at N={n}: rank {prog.rank} (busiest)",
        "launches": len(rows),
        "dram_bytes_per_step": sum(r["read"] + r["write"] for r in rows),
        "dram_bytes_per_launch": [r["read"] + r["write"] for r in rows],
        "algorithmic_bytes_per_step": algorithmic_bytes(prog),
        "capture": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                   f"-k regex:attn_fwd_kernel python tools/traffic_capture.py {n} (cold cache, serialised launches)",
    }
    with open(OUT, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc[f"n{n}"]))


if __name__ == "__main__":
    if sys.argv[1] == "--collect":
        collect(int(sys.argv[2]), sys.argv[3])
    else:
        run(int(sys.argv[1]))
