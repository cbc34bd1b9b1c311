"""SASS instruction counts of the hot kernels in libtdc.so (cuobjdump -sass): total instructions,
code bytes and the Blackwell-specific opcodes that prove the tcgen05 / TMA / TMEM paths.
Usage: python scripts/sass_counts.py > profiles/r02_sass_counts.txt"""
import collections, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2211_03715_b200", "libtdc.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
HOT = ["tdc_bf_layer_tm_kernel", "tdc_bf_core2_kernel", "tdc_bf_core_kernelILb0ELi0ELb0E", "tdc_bf_core_kernelILb1ELi0ELb0E",
       "tdc_bf_gemm_kernelILb1ELi0ELb1E", "tdc_bf_gemm_kernelILb0ELi0ELb0E", "tdc_sgemm_taps_kernel"]
OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM", "SYNCS", "FFMA", "HMMA"]
cur, stats = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        stats[cur] = collections.Counter()
        continue
    if cur and re.search(r"/\*[0-9a-f]{4,}\*/", line):
        stats[cur]["_n"] += 1
        op = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if op:
            for o in OPS:
                if op.group(1).startswith(o):
                    stats[cur][o] += 1
print("# cuobjdump -sass paper_2211_03715_b200/libtdc.so: hot kernels (static counts)")
print(f"{'kernel':60s} {'instr':>6s} {'bytes':>7s} " + " ".join(f"{o:>7s}" for o in OPS))
for name, c in stats.items():
    if not any(h in name for h in HOT):
        continue
    short = re.sub(r"^_ZN3tdc\d+", "", name)[:58]
    print(f"{short:60s} {c['_n']:6d} {16 * c['_n']:7d} " + " ".join(f"{c[o]:7d}" for o in OPS))
