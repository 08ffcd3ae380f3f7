from paper_2210_09147_b200.partime.pipeline import Pipeline, Stage  # noqa: F401
