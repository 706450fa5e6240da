"""Independent closed forms and quadratures that pin the oracle (not oracle code)."""
