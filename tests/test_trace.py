"""Measured-trace export uses the reference's Chrome trace schema
(simulator.py:365-382): X events, us timestamps, pid = node, tid = rank.stream."""
from paper_2509_21841_b200 import trace


def test_chrome_schema_matches_reference_layout():
    evs = [{"rank": 3, "stream": "compute", "start": 0.002, "duration": 0.001, "kind": "local.attn",
            "payload": {"pairs": 10}},
           {"rank": 1, "stream": "intra-comm", "start": 0.001, "duration": 0.0005, "kind": "kv.send",
            "payload": {"dst": 2, "round": 0, "ring": 0, "tokens": 5}}]
    doc = trace.to_chrome(evs, gpus_per_node=2)
    assert doc["displayTimeUnit"] == "ms"
    first, second = doc["traceEvents"]
    assert first["name"] == "kv.send" and first["ph"] == "X"
    assert first["ts"] == 1000.0 and first["dur"] == 500.0
    assert first["pid"] == 0 and first["tid"] == "1.intra-comm"
    assert list(first["args"]) == sorted(first["args"])
    assert second["pid"] == 1 and second["tid"] == "3.compute"
