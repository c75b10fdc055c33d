"""Ring-hop bandwidth from a tools/trace_layer.py trace: per hop and overall
(sum of bytes / sum of copy durations), python tools/hop_rates.py TRACE.json"""
import json
import sys

ev = json.load(open(sys.argv[1]))["traceEvents"]
hops = [e for e in ev if e["name"] == "kv.send"]
for e in hops:
    a = e["args"]
    print(f"{e['tid']:>14s} ring {a['ring']} round {a['round']}: {a['bytes'] / 1e6:7.1f} MB in "
          f"{e['dur'] / 1e3:6.3f} ms = {a['bytes'] / (e['dur'] * 1e-6) / 1e9:6.1f} GB/s")
tb = sum(e["args"]["bytes"] for e in hops)
td = sum(e["dur"] for e in hops)
print(f"{len(hops)} hops, {tb / 1e9:.2f} GB, overall {tb / (td * 1e-6) / 1e9:.1f} GB/s")
