"""Registration harness: INI run configuration
(``runconfig``), deterministic CSV / text reports (``report``) and the CLI the
reference declares (``pyproject.toml:20``, ``SPEC.md:514``) but never shipped
(``cli``: ``register | synthesize | check-derivatives | report``).
Host-side plumbing around the B200 solver; no numerics of its own."""
