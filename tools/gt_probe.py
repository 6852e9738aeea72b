import sys, os, torch
sys.path.insert(0,'.')
from paper_2109_13176_b200 import GvomMap, LAYERS, synth
w=synth.workload(1); f=w.frames[0]; dev=torch.device('cuda'); s=torch.cuda.Stream()
m=GvomMap(w.grid, max_points_per_frame=w.points_per_frame, stream=s)
scans=[(torch.from_numpy(x.points).to(dev), x.pose, x.rings) for x in f.scans]
with torch.cuda.stream(s):
    for mode in ("eager","graph"):
        m.set_timing(True, stages=["raycast"]); m.stage_times()
        for i in range(20):
            if mode=="graph": m.step(f.vehicle_xyz, scans)
            else:
                m.shift(f.vehicle_xyz); m.integrate_scan(scans); m.compute_maps(); m.export_layers()
        st=m.stage_times(); print(mode, st.get('raycast'), m.graph_stats())
