"""The synthetic workloads of BASELINE.json's five configs.

All batches come from the seeded sampler (``batch.sample_batch``), which is
draw-for-draw identical to the reference sampler, so every config names the
same sequences in the reference and here.
"""

from __future__ import annotations

from .batch import LengthDistribution, SequenceBatch, preset, sample_batch
from .cluster import ClusterSpec, single_box

# Llama-3-8B attention layer
HQ, HKV, HEAD_DIM, HIDDEN = 32, 8, 128, 4096


def github_le128k() -> LengthDistribution:
    """github mixture with the (128K, 256K] bin dropped and renormalised."""
    return LengthDistribution.normalized([b for b in preset("github").bins if b[1] <= 131072])


def c1_batch() -> SequenceBatch:
    """Tiny oracle config: lengths floor(exp(U(log 32, log 513))), rng seed 2."""
    return SequenceBatch(tuple(enumerate([66, 73, 306, 41, 169, 241, 53, 37])))


def c1_cluster() -> ClusterSpec:
    return ClusterSpec(num_nodes=1, gpus_per_node=2, token_capacity=497, inv_bw_intra=1.0, inv_bw_inter=1.0)


def c2_batch(preset_name: str = "github", seed: int = 0, total: int = 65536) -> SequenceBatch:
    """64K-token varlen batch, all GPU-local on one B200."""
    return sample_batch(preset(preset_name), total, seed)


def c3_batch(gpus: int, per_gpu: int = 65536, long_len: int = 131072, seed: int = 1) -> SequenceBatch:
    """Weak-scaling long-context mixture: one 128K sequence plus a github<=128K
    sample filling T = per_gpu * gpus tokens (ids shifted by one)."""
    total = per_gpu * gpus
    head = min(long_len, total)
    rest = sample_batch(github_le128k(), total - head, seed) if total > head else SequenceBatch(())
    return SequenceBatch(((0, head),) + tuple((sid + 1, n) for sid, n in rest.sequences))


def c4_batch(total: int = 262144, seed: int = 1) -> SequenceBatch:
    """256K-token github<=128K batch for the remap / full-block configs."""
    return sample_batch(github_le128k(), total, seed)


def cluster_for(batch: SequenceBatch, gpus: int) -> ClusterSpec:
    return single_box(gpus, batch.total_tokens)
