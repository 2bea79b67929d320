"""Summarise `ptxas -v` output: kernel template id, registers, stack, spills."""
import re
import subprocess
import sys

lines = sys.stdin.read().splitlines()
cur = None
for ln in lines:
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        name = m.group(1)
        k = re.search(r"\d+([a-z_]+kernel)(I.*?EEv)?", name)
        cur = (k.group(1) + (k.group(2) or "")) if k else name[:60]
        continue
    m = re.search(r"Used (\d+) registers.*?(?:(\d+) bytes cumulative stack size)?", ln)
    if m and cur:
        st = re.search(r"(\d+) bytes cumulative stack", ln)
        print(f"{cur:45s} regs={m.group(1):>4s} stack={st.group(1) if st else 0}")
        cur = None
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and (m.group(1) != "0" or m.group(2) != "0"):
        print("   SPILL", ln.strip())
