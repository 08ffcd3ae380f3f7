"""Paper-facing API: partime.pipeline.Pipeline, partime.balancing."""
