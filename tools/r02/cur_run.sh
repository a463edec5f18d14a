# r29: PCIe copy roof with 1 / 2 / 4 streams per direction
timeout 300 python tools/r02/pcie_streams.py > gpurun_out/r29_pcie.log 2>&1
timeout 300 python tools/r02/pcie_streams.py >> gpurun_out/r29_pcie.log 2>&1
