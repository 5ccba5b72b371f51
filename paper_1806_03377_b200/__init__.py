"""B200-native PipeDream (arXiv 1806.03377) pipeline-parallel training runtime."""
