"""SparkNet data-parallel hot path, B200-native."""
