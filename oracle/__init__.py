"""CPU oracle for the SNP step (TEST INFRASTRUCTURE ONLY -- see snp_oracle.py)."""
