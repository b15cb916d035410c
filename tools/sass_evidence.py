"""Count Blackwell-relevant SASS mnemonics per kernel in libapex.so (no GPU needed).

    python tools/sass_evidence.py > profiles/r01_sass_evidence.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2506_03296_b200", "libapex.so")
MN = ("UTMALDG", "UBLKCP", "HMMA", "LDSM", "SYNCS", "FFMA", "MUFU.EX2", "LDS.128", "BAR.SYNC", "ATOMG", "LDG",
      "STG")
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
cur, cnt = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    for mn in MN:
        if re.search(r"\b" + re.escape(mn), line):
            cnt[cur][mn] += 1
print("# SASS mnemonic counts per kernel (cuobjdump -sass libapex.so, sm_100a).")
print("# UTMALDG = TMA tensor load, SYNCS = mbarrier ops, HMMA = mma.sync tensor-core MMA, LDSM = ldmatrix.\n")
for f, c in sorted(cnt.items()):
    if any(k in f for k in ("decode_kernel", "merge_kernel", "append_kernel", "apply_deltas", "synth_kernel")):
        print(f + "\n   " + ", ".join(f"{k}={v}" for k, v in sorted(c.items())))
