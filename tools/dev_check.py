"""Debug: run a preset through the device scheduler with the prescan-consumer self-check on."""
import ctypes as C
import os
import sys
sys.path.insert(0, ".")
os.environ.setdefault("CS_DEBUG_PRESCAN", "1")
import numpy as np
import paper_2605_27744_b200 as cb
from paper_2605_27744_b200._lib import lib
eng = cb.Engine(cb.preset_by_name(sys.argv[1]), policy=sys.argv[2], agent_capacity=1024)
eng.run()
buf = (C.c_uint64 * (16 * 1024))()
g = C.c_int(0)
lib().cs_pool_debug(lib().cs_engine_pool(eng.h), buf, 16 * 1024, C.byref(g))
d = np.array(buf[:16 * g.value + 192], dtype=np.uint64)
o = d[16 * g.value + 16:]
print("misses", int(o[0]))
for k in range(min(int(o[0]), 8)):
    r = o[1 + 6 * k:7 + 6 * k]
    print(f"slot {int(r[0])} lt {int(r[1])} agent {int(r[2]) >> 32:#x} inU {(int(r[2]) >> 1) & 1} touched {int(r[2]) & 1} "
          f"inPL {int(r[3]) & 0xffffffffff if int(r[3]) & 0xffffffffff != 0xffffffffff else -1} seq {int(r[4])} last_unpin seq {int(r[5]) >> 8} src {int(r[5]) & 255}")
o2 = d[16 * g.value + 72:]
print("tma/L2 mismatches", int(o2[0]))
for k in range(min(int(o2[0]), 8)):
    r = o2[1 + 6 * k:7 + 6 * k]
    print(f"slot {int(r[0])} tma_lt {int(r[1])} l2_lt {int(r[2])} tma_refs {int(r[3]) >> 32} l2_refs {int(r[3]) & 0xffffffff} cta {int(r[4]) & 0xffffffff} tile {int(r[4]) >> 32} verdict_seq {int(r[5])}")
print("poison seen", int(d[16 * g.value + 72]) if os.environ.get("CS_DEBUG_PRESCAN") == "6" else "-",
      "stale (mode 6)", int(d[16 * g.value + 128]) if os.environ.get("CS_DEBUG_PRESCAN") == "6" else "-")
print(eng.result()["hit_rate"])
