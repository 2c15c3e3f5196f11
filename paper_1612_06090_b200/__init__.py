"""B200-native SPH density / smoothing-length pass (drop-in for sphlab)."""
