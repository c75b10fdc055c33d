"""B200-native (sm_100a) per-layer hot path of Zeppelin (arXiv 2509.21841)."""
