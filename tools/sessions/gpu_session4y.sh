mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="hypercube3:4194304@spread:262144,hypercube3:4194304@spread:524288,hypercube3:4194304@cp:262144,hypercube3:4194304@cp:524288,hypercube3:4194304@static,hypercube3:4194304@ll128,hypercube3:4194304@mix:262144,hypercube3:4194304@ready:262144"
timeout 1200 $TR --nproc-per-node 4 --master-port 29931 tools/sweep.py --lowering balanced --steps 20 --cases "$C" --out gpurun_out/y4_h4m_G4.jsonl > gpurun_out/y4_h4m_G4.log 2>&1; echo "g4 rc=$?"
A2A_SPLIT_W=2 timeout 600 $TR --nproc-per-node 4 --master-port 29932 tools/sweep.py --lowering balanced --steps 20 --cases "hypercube3:4194304@static" --out gpurun_out/y4_h4m_w2_G4.jsonl > gpurun_out/y4_h4m_w2_G4.log 2>&1; echo "w2 rc=$?"
