#!/usr/bin/env python3
"""profiles/ncu_traffic.json (the `traffic` and `inst_per_voxel` of bench.py's roofline
object) from the ncu --set full summaries of one evidence run:
  python3 tools/ncu_traffic.py TAG"""
import json
import re
import sys

tag = sys.argv[1]
caps = {
    "c3/auto": ("c3", "1 launch of warp3d_cube_kernel<float,16,3,1,0,1,0,16>, C3 16x128x128x160"),
    "c4/auto": ("c4", "1 launch of warp3d_cube_kernel<float,8,3,1,0,1,0,16>, C4 512^3, "
                      "8-row tiles in bricks"),
    "resample/auto": ("resample", "1 launch of smooth_fused_kernel<2,4>, dense (warp3d_smooth3d), "
                                  "512^3 f32, sigma 2/3 voxel per axis"),
}
out = {}
for key, (w, what) in caps.items():
    path = f"profiles/round2/ncu_full_{w}_{tag}.txt"
    try:
        text = open(path).read()
    except OSError:
        continue
    mb = lambda n: float(re.search(rf"^{n}\s+([\d.]+) Mbyte", text, re.M).group(1)) * 1e6
    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    ipv = float(re.search(r"thread-instr/voxel ([\d.]+)", text).group(1))
    out[key] = {"dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
                "inst_per_voxel": ipv, "source": f"{path} (ncu --set full, {what})"}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
