"""B200-native device-placement REINFORCE hot path (arXiv 1706.04972)."""
