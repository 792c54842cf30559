import sys, re, collections, subprocess
cub, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
cnt = collections.Counter(); cur = None; infn = False
for line in out.splitlines():
    if line.startswith("//---") and ".text." in line:
        infn = fn in line
    if not infn: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', line): cnt[cur] += 1
tot = sum(cnt.values()); print('total', tot)
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30): print(v, k)
