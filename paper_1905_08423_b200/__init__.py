"""B200-native C = P^T A P (placeholder init; filled in below)."""
