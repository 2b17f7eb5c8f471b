# 4-GPU probe: NVLink ceiling of all-to-all-shaped push patterns + NVML counter fields
mkdir -p gpurun_out
timeout 600 python tools/nvlink_a2a_probe.py --gpus 4 > gpurun_out/p4_a2a_probe.json 2> gpurun_out/p4_a2a_probe.err; echo "probe4 rc=$?"
timeout 600 python tools/nvlink_a2a_probe.py --gpus 2 > gpurun_out/p4_a2a_probe_g2.json 2> gpurun_out/p4_a2a_probe_g2.err; echo "probe2 rc=$?"
nvidia-smi nvlink -gt d > gpurun_out/p4_smi_nvlink_gt.txt 2>&1; echo "smi rc=$?"
nvidia-smi nvlink -s -i 0 > gpurun_out/p4_smi_nvlink_s.txt 2>&1
