"""Bundled topology documents (reference ``pkg/src/scalesim/presets.py``) plus B200 hosts.

The reference's evaluation clusters and cloud instance types are reproduced
value for value from one table.  The ``b200-*`` rows describe HGX B200 boxes:
8 GPUs per host on NVLink 5 / NVSwitch at 900 GB/s per direction (7200 Gbps),
a PCIe Gen5 x16 host link (64 GB/s nominal = 512 Gbps), 400 Gbps ConnectX-7
per GPU between hosts and an NVMe share per GPU.
"""

#  name                   hosts gpus  intra     intra_gbps inter_gbps host_gpu ssd_gpu
_TABLE = (
    ("cluster-A",            4, 8, "nvlink", 1600.0, 100.0, 128.0, 10.0),
    ("cluster-B",            2, 8, "pcie",    256.0, 100.0, 128.0, 10.0),
    ("a2-ultragpu-8g",       2, 8, "nvlink", 1600.0,  12.5, 128.0, 2.58),
    ("p4d.24xlarge",         2, 8, "nvlink", 1600.0, 100.0, 128.0, 2.31),
    ("ml.hpcpni2.28xlarge",  2, 8, "pcie",    256.0, 100.0, 128.0, 4.0),
    ("p4de.24xlarge",        2, 8, "nvlink", 1600.0, 100.0, 128.0, 2.31),
    ("a3-highgpu-8g",        2, 8, "nvlink", 1600.0, 100.0, 128.0, 6.09),
    ("a3-megagpu-8g",        2, 8, "nvlink", 1600.0, 200.0, 128.0, 6.09),
    ("p5.48xlarge",          2, 8, "nvlink", 1600.0, 400.0, 128.0, 9.8),
    ("b200-hgx",             1, 8, "nvlink", 7200.0, 400.0, 512.0, 50.0),
    ("b200-hgx-2x8",         2, 8, "nvlink", 7200.0, 400.0, 512.0, 50.0),
)


def topology_document(num_hosts: int, gpus_per_host: int, intra_kind: str,
                      intra_gbps: float, inter_gbps: float, host_gpu_gbps: float,
                      ssd_gpu_gbps: float) -> dict:
    """A homogeneous cluster document in the ``load_topology`` schema."""
    hosts = [dict(id=h, gpus=gpus_per_host, host_gpu_gbps=host_gpu_gbps,
                  ssd_gpu_gbps=ssd_gpu_gbps) for h in range(num_hosts)]
    return dict(hosts=hosts, intra=dict(kind=intra_kind, gbps=intra_gbps),
                inter=dict(gbps=inter_gbps))


PRESETS: dict[str, dict] = {row[0]: topology_document(*row[1:]) for row in _TABLE}
