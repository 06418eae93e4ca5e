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
    try:
        info = pynvml.c_nvmlGpuFabricInfoV_t()
        info.version = pynvml.nvmlGpuFabricInfo_v3 if hasattr(pynvml, "nvmlGpuFabricInfo_v3") \
            else pynvml.nvmlGpuFabricInfo_v2
        pynvml.nvmlDeviceGetGpuFabricInfoV(h, info)
        states = {0: "NOT_SUPPORTED", 1: "NOT_STARTED", 2: "IN_PROGRESS", 3: "COMPLETED"}
        out["fabric"] = {"state": states.get(info.state, info.state), "status": int(info.status),
                         "clique_id": int(info.cliqueId),
                         "cluster_uuid": bytes(info.clusterUuid).hex()}
    except Exception as e:  # older NVML: the v1 query
        try:
            f = pynvml.nvmlDeviceGetGpuFabricInfo(h)
            out["fabric"] = {"state": int(f.state), "status": int(f.status)}
        except Exception as e2:
            out["fabric_error"] = f"{e}; {e2}"
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
