"""pipestream.cli: the console entry point the reference declares
(pkg/pyproject.toml:21-22, `pipestream = "pipestream.cli:main"`)."""
from paper_2210_09147_b200.cli import main  # noqa: F401

if __name__ == "__main__":
    raise SystemExit(main())
