"""Per-kernel registers / stack (spills) of a built object, from cuobjdump -res-usage.

    python tools/resusage.py paper_2110_05722_b200/lib/obj/layernorm.o [name-filter]
"""

import re
import subprocess
import sys


def main():
    obj = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["cuobjdump", "-res-usage", obj], capture_output=True, text=True).stdout
    names = subprocess.run(["c++filt"], input="\n".join(re.findall(r"Function (\S+):", out)),
                           capture_output=True, text=True).stdout.splitlines()
    stats = re.findall(r"REG:(\d+) STACK:(\d+) SHARED:(\d+)", out)
    for name, (reg, stack, shared) in zip(names, stats):
        if filt in name:
            short = re.sub(r"\(.*\)$", "", name).replace("ls2::", "")
            flag = "  <-- spills" if int(stack) > 16 else ""
            print(f"REG {reg:>3} STACK {stack:>4} SMEM {shared:>5}  {short}{flag}")


if __name__ == "__main__":
    main()
