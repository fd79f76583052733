"""TEST INFRASTRUCTURE ONLY — parity checkers (see oracle/oracle.py).  Never
imported by the product package paper_2605_02171_b200/."""
