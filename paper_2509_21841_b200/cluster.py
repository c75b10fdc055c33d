"""Cluster description consumed by the planner.

Mirrors the reference ``ClusterSpec`` (``topology.py:22-64``): N nodes x P GPUs
with a per-rank token capacity L; the two inverse-bandwidth coefficients only
feed the remap cost matrix.  Cost-model calibration knobs
(``CostCoefficients``, zone boundaries, config files) are out of scope here:
the partitioner never reads them.
"""

from __future__ import annotations

from dataclasses import dataclass

# K+V bytes of one KV token in the reference's cost model (topology.py:14-15).
KV_BYTES_PER_TOKEN = 16384


class ConfigError(ValueError):
    """Invalid cluster parameters (reference ``topology.py:18``)."""


@dataclass(frozen=True)
class ClusterSpec:
    num_nodes: int
    gpus_per_node: int
    token_capacity: int
    inv_bw_intra: float
    inv_bw_inter: float
    nics_per_node: int = 1
    backward_multiplier: float = 2.0

    def __post_init__(self) -> None:
        checks = (
            (self.num_nodes >= 1, "num_nodes must be >= 1"),
            (self.gpus_per_node >= 1, "gpus_per_node must be >= 1"),
            (self.token_capacity >= 1, "token_capacity must be >= 1"),
            (self.nics_per_node >= 1, "nics_per_node must be >= 1"),
            (self.inv_bw_intra > 0, "inv_bw_intra must be > 0"),
            (self.inv_bw_inter >= self.inv_bw_intra, "inv_bw_inter must be >= inv_bw_intra"),
            (self.backward_multiplier >= 0, "backward_multiplier must be >= 0"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)

    @property
    def num_ranks(self) -> int:
        return self.num_nodes * self.gpus_per_node

    def node_of(self, rank: int) -> int:
        return rank // self.gpus_per_node

    def ranks_of_node(self, node: int) -> range:
        first = node * self.gpus_per_node
        return range(first, first + self.gpus_per_node)


def single_box(gpus: int, total_tokens: int, slack: float = 1.05,
               link_bytes_per_s: float = 900e9, kv_bytes_per_token: int = 4096) -> ClusterSpec:
    """One NVSwitch box of ``gpus`` B200s: N=1, P=gpus, L=ceil(slack*T/G)
    (exact capacity is infeasible for most single-node batches; 5% slack is
    always feasible on the measured presets)."""
    cap = max(1, -(-int(round(slack * 1000)) * total_tokens // (1000 * gpus)))
    inv = kv_bytes_per_token / link_bytes_per_s
    return ClusterSpec(num_nodes=1, gpus_per_node=gpus, token_capacity=cap,
                       inv_bw_intra=inv, inv_bw_inter=inv)
