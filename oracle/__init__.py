"""Test-only CPU oracle (see ils_oracle.py header). Never imported by the product."""
