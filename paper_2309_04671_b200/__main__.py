"""``python -m paper_2309_04671_b200 <command> ...`` — the reference CLI on B200.

Runs the reference's own command line (``stencilkit.cli.main``: ``run``,
``compile``, ``inspect``, ``simulate``, ``diff``) with the drop-in installed
(:func:`.integrate.install`), so ``run --backend gpu`` (cli.py:246-283)
executes the bound target on the device: same flags, same STG1 output
files, same ``--oracle`` report and exit codes (0 ok, 1 diagnostics, 2
tolerance failure, 3 internal error; cli.py:393-410).  One extra flag,
``--precision fast|exact`` (default exact; env ``STKB_PRECISION``), picks the
device arithmetic; it is removed before the reference parses the rest.
"""

from __future__ import annotations

import sys

from . import front
from .integrate import install


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    precision = None
    if "--precision" in argv:
        i = argv.index("--precision")
        if i + 1 >= len(argv) or argv[i + 1] not in ("fast", "exact"):
            print("error: --precision expects fast or exact", file=sys.stderr)
            return 1
        precision = argv[i + 1]
        del argv[i:i + 2]
    install(precision)
    return front.module("cli").main(argv)


if __name__ == "__main__":
    sys.exit(main())
