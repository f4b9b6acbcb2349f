"""B200-native LB-BSP iteration hot path (arXiv 1806.02508)."""
