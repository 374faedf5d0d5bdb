"""B200-native FairBatching per-iteration scheduling hot path (fbsim drop-in)."""
