import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate", "Grid Size",
        "Dynamic Shared Memory Per Block", "SM Active Cycles", "Elapsed Cycles", "Waves Per SM",
        "Compute (SM) Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput")
for row in r[1:]:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in keep:
        print(f"{d.get('Kernel Name','')[:30]:30s} {d['Metric Name']:38s} {d['Metric Value']} {d.get('Metric Unit','')}")
