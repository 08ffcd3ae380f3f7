from paper_2210_09147_b200.partime.balancing import balance_pipeline_partitions, balance_model  # noqa: F401
