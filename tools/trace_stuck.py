"""Where a stalled sweep stopped (trace written with TIB_TRACE after a watchdog
abort): tasks claimed but never finished (with the dependencies they list),
tasks pushed but never claimed, and each chain's last recorded step."""
import sys

import numpy as np

from trace_report import label, load, where

d = load(sys.argv[1])
tasks, deps, rec, nq0 = d["tasks"], d["deps"], d["rec"], d["nq0"]
claimed = (rec[:, 0] > 0) & (rec[:, 2] == 0)
pushed_only = (rec[:, 1] > 0) & (rec[:, 0] == 0)
done = rec[:, 2] > 0
print(f"tasks {len(tasks)}: done {done.sum()}, claimed-not-done {claimed.sum()}, pushed-not-claimed {pushed_only.sum()}")
for name, m in (("claimed, not done", claimed), ("pushed, not claimed", pushed_only)):
    idx = np.nonzero(m)[0][:25]
    print(name)
    for ti in idx:
        t = tasks[ti % len(tasks)]
        dl = deps[t["dep_begin"]: t["dep_begin"] + t["dep_count"] + t["dep2_count"]]
        print(f"  task {ti} {label(t, ti < nq0)} {where(t, d['tiles'], d['bp'])} poll {t['poll']} "
              f"deps {[(int(x['counter']), int(x['value'])) for x in dl][:8]} dep2 {int(t['dep2_count'])}")
ch = d["chain"]
if len(ch):
    started = np.nonzero(ch[:, 0] > 0)[0]
    print("chain steps recorded:", len(started), "of", len(ch), "last index", started.max() if len(started) else None)
    ct = d["chain_tasks"]
    for s in started[-4:]:
        t = ct[s]
        dl = deps[t["dep_begin"]: t["dep_begin"] + t["dep_count"] + t["dep2_count"]]
        print(f"  step {s} rec {ch[s].tolist()} deps {[(int(x['counter']), int(x['value'])) for x in dl][:6]}")

# Which never-run tasks had every first-phase dependency produced (a lost
# push), and which dependencies block the others.  Counts each counter's
# signals from the tasks and chain steps that finished.
sigs = d["sigs"]
cnt = {}
def add(t):
    for s in sigs[t["sig_begin"]: t["sig_begin"] + t["sig_count"]].tolist():
        cnt[s] = cnt.get(s, 0) + 1
nt = len(tasks)
for i in np.nonzero(done)[0]:
    t = tasks[i % nt]
    if t["kind"] == 2 and (int(t["aux1"]) >> 8) != (int(t["aux1"]) & 255) - 1:
        pass  # split parts: the group signals once (counted below per group)
    else:
        add(t)
# split groups: the reducer (last arrival) signals; count a group once when all its parts finished
groups = {}
for i in range(nt):
    t = tasks[i]
    if t["kind"] == 2:
        groups.setdefault(int(t["aux0"]), []).append(i)
for g, parts in groups.items():
    if all(done[p] for p in parts):
        add(tasks[parts[-1]])  # (the last part in plan order carries the same signals)
for s in np.nonzero(ch[:, 2] > 0)[0] if len(ch) else []:
    add(d["chain_tasks"][s])
never = np.nonzero(~done & ~claimed)[0]
lost, blocked = [], {}
for ti in never:
    t = tasks[ti % nt]
    dl = deps[t["dep_begin"]: t["dep_begin"] + t["dep_count"]]
    miss = [(int(x["counter"]), int(x["value"]), cnt.get(int(x["counter"]), 0)) for x in dl if cnt.get(int(x["counter"]), 0) < int(x["value"])]
    if not miss:
        lost.append(ti)
    else:
        for m in miss:
            blocked[m[0]] = blocked.get(m[0], 0) + 1
print("never-run tasks", len(never), "with every first-phase dependency produced (lost push):", len(lost))
for ti in lost[:15]:
    t = tasks[ti % nt]
    print(f"  lost task {ti} {label(t, ti < nq0)} {where(t, d['tiles'], d['bp'])} poll {t['poll']}")
top = sorted(blocked.items(), key=lambda kv: -kv[1])[:10]
print("most-missed counters (counter: tasks blocked):", top)
