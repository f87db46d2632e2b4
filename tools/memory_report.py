"""Print the storage accounting (Eq 6.1-6.3, fmg_memory_model) of C1-C5 as a
markdown table (host only; no GPU needed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_19036_b200 as P
from fmg_inputs import CONFIGS

print("| config | n_L | ú bits/DoF | r bits/DoF | Eq 6.1 ú sum / bound | exponents fixed / streaming "
      "| Eq 6.2 u,t / Eq 6.3 z (bits/DoF) | FP64 temporaries (B/DoF) | sections (B/DoF) |")
print("|---|---|---|---|---|---|---|---|---|")
for k in sorted(CONFIGS):
    c = CONFIGS[k]
    m = P.memory_model(c["dim"], c["p"], c["levels"])
    n = m["unknowns"]
    print(f"| {k} | {n:.3g} | {m['u_mantissa_bits']/n:.2f} | {m['r_mantissa_bits']/n:.2f} "
          f"| {m['eq61_u']/n:.2f} / {m['eq61_u_bound']/n:.2f} "
          f"| {m['exponent_bits_fixed']/n:.3f} / {m['exponent_bits_streaming']/n:.1e} "
          f"| {m['eq62_ut_bits']/n:.3f} / {m['eq63_z_bits']/n:.3f} | {m['fp64_temporary_bytes']/n:.1f} "
          f"| {m['section_bytes']/n:.2f} |")
