#!/bin/bash
# ncu --set full of the force kernel on the interleaved list (and the plain one), isolated
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1
python tools/one_force.py il > gpurun_out/u_plain_run.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_force -s 1 -c 1 -o gpurun_out/u_force_il python tools/one_force.py il > gpurun_out/u_ncu_il.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_force -s 1 -c 1 -o gpurun_out/u_force_plain python tools/one_force.py plain > gpurun_out/u_ncu_plain.log 2>&1
ncu --set full --clock-control none -k regex:k_gather_probe -s 1 -c 1 -o gpurun_out/u_probe_il python -c "
import os,sys,torch; sys.path.insert(0,os.getcwd()); import lj_inputs; from paper_1806_05713_b200 import lj
w=lj_inputs.config(4); g=lj.geom(w.L,w.rc,w.rs); q0=lj.pack_aos4(torch.from_numpy(w.q).cuda()); q=lj.permute_rows(q0,lj.cell_order(q0,g))
lst=lj.ListBuilder(w.n,g,False,device='cuda',padded=True,interleaved=True).build(q); s=torch.zeros(4,dtype=torch.float64,device='cuda')
[lj.gather_probe(q,lst,4|768,s) for _ in range(3)]; torch.cuda.synchronize()" > gpurun_out/u_ncu_probe.log 2>&1
