"""Test-infrastructure oracle package (see oracle/oracle.py).  Not part of the
product; never imported by paper_2407_00019_b200."""
