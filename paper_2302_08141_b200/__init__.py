"""B200-native executor for Rhino-partitioned tensor programs (arXiv 2302.08141)."""
