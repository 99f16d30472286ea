"""B200-native SN-like DLR hot path."""
