#!/bin/bash
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1
timeout 300 python tools/pcie_probe.py > gpurun_out/x_pcie.log 2>&1
nvidia-smi -q | grep -i -A4 "PCI\b\|Link Width\|Link Gen\|GPU Link" > gpurun_out/x_pci_info.log 2>&1
nvidia-smi topo -m >> gpurun_out/x_pci_info.log 2>&1
