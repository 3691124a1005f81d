"""Static SASS opcode counts of the step kernels in the built library
(cuobjdump -sass) and, where an ncu --set full capture exists, the dynamic
(executed) instruction mix -> profiles/r02_sass.md (scratch tool)."""
import collections, csv, io, re, subprocess, sys
LIB = "/root/repo/paper_2409_05205_b200/libhe_rotfree.so"
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if cur and m:
        funcs[cur][m.group(2)] += 1
# the instances the config-4 / config-5 steps launch (profiles/launches_r02.csv)
want = [("k_ntt_fwd_dp_s1<2,14,3,2,8,16,16> (forward NTT, s = 8)", "_Z15k_ntt_fwd_dp_s1ILi2ELi14ELi3ELi2ELi8ELi16ELi16EE"),
        ("k_mac_imma<2,5,16,16,16,4,1,3> (MAC, K = 16, s = 8)", "_Z10k_mac_immaILi2ELi5ELi16ELi16ELi16ELi4ELi1ELi3EE"),
        ("k_intt_scatter<1,14,3,2,2184,4,8,34,32,1,3> (INTT + scatter, s = 8)", "_Z14k_intt_scatterILb1ELi14ELi3ELi2ELi2184ELi4ELi8ELi34ELi32ELi1ELi3EE"),
        ("k_intt_rows<2,14,5,8,546,4,32,1> (INTT + rows, s = 32)", "_Z11k_intt_rowsILi2ELi14ELi5ELi8ELi546ELi4ELi32ELi1EE"),
        ("k_ntt_fwd_cols<2,7,5,137> (forward NTT, column form: s = 128, config 5)", "_Z14k_ntt_fwd_colsILi2ELi7ELi5ELi137EE"),
        ("k_mac_tc<1,true> (tcgen05 MAC with TMA staging, B >= 128, config 5)", "_Z8k_mac_tcILi1ELb1EE")]
def find(prefix):
    for f in funcs:
        if f.startswith(prefix):
            return f
    return None
lines = ["# Round 2: SASS of the step kernels (sm_100a, `cuobjdump -sass` of libhe_rotfree.so)", "",
         "Static instruction counts per opcode (top 14); the tensor-core and FP64 opcodes show",
         "which pipe each kernel is built on (IMMA = mma.sync int8, UTCMMA / UTC* = tcgen05,",
         "DFMA/DADD/DMUL = the FP64 modular arithmetic, UBLKCP = TMA bulk copy).", ""]
for i, (title, name) in enumerate(want):
    name = find(name)
    c = funcs.get(name)
    if not c:
        lines.append(f"## {title}\n\n(not found)\n")
        continue
    tot = sum(c.values())
    lines.append(f"## {title}\n\n`{name}` -- {tot} instructions\n")
    lines.append("| opcode | count |\n|---|---|")
    for op, n in c.most_common(14):
        lines.append(f"| {op} | {n} |")
    key = {op: c[op] for op in ("IMMA", "UTCIMMA", "UTMALDG", "UBLKCP", "LDGSTS", "DFMA", "SYNCS")
           if c.get(op)}
    lines.append("")
    lines.append("pipe-defining opcodes: " + ", ".join(f"{k} {v}" for k, v in key.items()))
    lines.append("")
open("/root/repo/profiles/r02_sass.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines)[:1500])
