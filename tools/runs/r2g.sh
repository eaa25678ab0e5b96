python tools/diag_moe.py
