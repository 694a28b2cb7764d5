"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path used as
the parity checker (tests/, __graft_entry__.smoke) and as bench.py's CPU
baseline arm. Never imported by the product package."""
