"""Import shim for the paper's module path: `from partime.pipeline import Pipeline`."""
