"""Static SASS instruction count per source line of one kernel (nvdisasm -g)."""
import collections, re, subprocess, sys
cubin, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur = None; cnt = collections.Counter(); inside = False
for line in out.splitlines():
    if line.startswith(".text."):
        inside = fn in line
        continue
    if not inside: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split("/")[-1], int(m.group(2))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', line): cnt[cur] += 1
print("total", sum(cnt.values()))
for k, v in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30): print(v, k)
