"""Why is NVLink-SHARP multicast (multimem.*) unavailable on this lease?
Prints one JSON object: the CUDA multicast attribute, NVML's GPU fabric state
(the NVSwitch fabric manager registers each GPU into an NVLink partition; a
multicast object can only span GPUs registered in one), the visible GPU count,
and the result of tools/nvls_probe.cu's cuMulticastCreate attempts."""
import json
import subprocess

out = {}
try:
    import pynvml

    pynvml.nvmlInit()
    out["visible_gpus"] = pynvml.nvmlDeviceGetCount()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    out["name"] = pynvml.nvmlDeviceGetName(h)
    # (the struct-versioned NVML fabric query crashed this image's pynvml: the
    # fabric state is read from `nvidia-smi -q` below instead)
    try:
        out["nvlink_active_links"] = sum(
            1 for i in range(18)
            if pynvml.nvmlDeviceGetNvLinkState(h, i) == pynvml.NVML_FEATURE_ENABLED)
    except Exception as e:
        out["nvlink_error"] = str(e)
except Exception as e:
    out["nvml_error"] = str(e)
try:
    q = subprocess.run(["nvidia-smi", "-q"], capture_output=True, text=True, timeout=60).stdout
    lines = q.splitlines()
    for i, line in enumerate(lines):
        if line.strip().startswith("Fabric"):
            out["nvidia_smi_fabric"] = [x.strip() for x in lines[i:i + 8]]
            break
except Exception as e:
    out["nvidia_smi_error"] = str(e)
print(json.dumps(out))
