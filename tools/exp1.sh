mkdir -p gpurun_out
timeout 120 python -c "
import paper_2601_21622_b200 as sd, torch
for a in [(64,5,32000,1.0,torch.float32),(128,7,128256,1.0,torch.float32),(128,7,128256,1.0,torch.bfloat16)]:
    print(a[:4], a[4], sd.plan(*a))
" > gpurun_out/plan.log 2>&1
for kb in 32 128; do
STARSD_CTA_KB=$kb timeout 120 python -c "
import paper_2601_21622_b200 as sd, torch
for a in [(64,5,32000,1.0,torch.float32),(128,7,128256,1.0,torch.float32)]:
    print($kb, a[:4], a[4], sd.plan(*a))
" >> gpurun_out/plan.log 2>&1
STARSD_CTA_KB=$kb timeout 300 python bench.py --no-cpu --no-e2e --steps 300 > gpurun_out/e_c2_$kb.json 2>&1
STARSD_CTA_KB=$kb timeout 300 python bench.py --config c3 --no-cpu --no-e2e --steps 200 > gpurun_out/e_c3_$kb.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_verify_cluster" -s 6 -c 1 -f -o gpurun_out/cl_c3 python tools/profile_run.py --config c3 --calls 8 > gpurun_out/ncu_cl_c3.log 2>&1
