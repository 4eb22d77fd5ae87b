"""B200-native exhaustive Gray-code search for the L_d norms of arXiv 2503.21596."""
