import re, csv, sys, subprocess, collections
dis, rep, kern = sys.argv[1], sys.argv[2], sys.argv[3]
import os; src = open(os.environ.get('SRC','/root/repo/paper_1910_11872_b200/csrc/demod_kernel.cuh')).read().splitlines()
# parse disassembly of the kernel
lines = open(dis).read().splitlines()
start = None
for i, l in enumerate(lines):
    if l.startswith('.text.' + kern + ':'):
        start = i; break
chain = []
addr2 = {}
for l in lines[start+1:]:
    if l.startswith('//----') or l.startswith('.text.'):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        rest = m.group(3)
        ch = [(m.group(1), int(m.group(2)))] + [(a, int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', rest)]
        chain = ch
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m:
        addr2[int(m.group(1), 16)] = (chain, m.group(2))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr)]
base = int(data[0][ix['Address']], 16)
by_outer = collections.Counter(); by_inner = collections.Counter(); tot = 0
for r in data:
    a = int(r[ix['Address']], 16) - base
    ex = int(r[ix[os.environ.get('COL', 'Thread Instructions Executed')]] or 0)
    tot += ex
    ch = addr2.get(a, ([], ''))[0]
    kl = [ln for f, ln in ch if f.endswith(os.path.basename(os.environ.get('SRC','demod_kernel.cuh')))]
    outer = kl[-1] if kl else -1
    by_outer[outer] += ex
    # second level: first kernel-file line in the chain that is > 80 (inside a device function body)
    inner = kl[-2] if len(kl) >= 2 else outer
    by_inner[(outer, inner)] += ex
print("total thread-instructions", tot)
for ln, v in sorted(by_outer.items(), key=lambda x: -x[1])[:25]:
    print(f"{v/tot*100:5.1f}%  L{ln:4d}: {src[ln-1].strip()[:90] if ln>0 else ''}")
print("--- inner (within helpers)")
for (o, i), v in sorted(by_inner.items(), key=lambda x: -x[1])[:25]:
    print(f"{v/tot*100:5.1f}%  L{o}->L{i}: {src[i-1].strip()[:80] if i>0 else ''}")
