"""Physical constants (reading C8).  gamma>0 is only named at P:187; hbar default P:370."""
import math

GAMMA = 1.7595e11            # rad s^-1 T^-1
MU0 = 4e-7 * math.pi         # T m A^-1
HBAR = 1.05457182e-34        # J s (the HBAR built-in default)
KB = 1.380649e-23            # J K^-1 (SI exact; the thermal field, reading C-TH)
