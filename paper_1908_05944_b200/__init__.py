"""B200-native alpha-complex hot path (drop-in for alphax.compute_alpha_complex)."""
