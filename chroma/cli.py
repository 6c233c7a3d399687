"""Drop-in module path: `chroma.cli` (pyproject.toml:16 console script chroma.cli:main)
-> paper_2107_00075_b200.cli."""
from paper_2107_00075_b200.cli import *  # noqa: F401,F403
from paper_2107_00075_b200.cli import main  # noqa: F401

if __name__ == "__main__":
    import sys
    sys.exit(main())
