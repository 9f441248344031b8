"""B200-native GPU-IM process mapping (drop-in for promap.pipelines.integrated_map)."""
