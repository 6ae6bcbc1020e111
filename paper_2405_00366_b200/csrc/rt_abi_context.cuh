// rt_abi_context.cuh -- part of the single runtime TU (runtime.cu includes the parts in
// order): C ABI: context lifecycle and options.
#pragma once

extern "C" {

int cimcs_create(int32_t device, int32_t dtype, cimcs_ctx** out) {
    if (!out) return fail(CIMCS_INPUT_ERROR, "null out");
    if (dtype != CIMCS_F32 && dtype != CIMCS_F64) return fail(CIMCS_CONFIG_ERROR, "bad dtype");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(CIMCS_CONFIG_ERROR, "bad device");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(CIMCS_CUDA_ERROR, "libcimcs_gpu is built for sm_100a (B200) only");
    auto* c = new cimcs_ctx();
    c->num_sms = prop.multiProcessorCount;
    c->device = device;
    c->dtype = dtype;
    c->host_threads = std::max(1u, std::thread::hardware_concurrency());
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return fail(CIMCS_CUDA_ERROR, "stream create failed");
    }
    if (dalloc(c, &c->alt, sizeof(AltParams)) || dalloc(c, &c->err, 16)) {
        delete c;
        return CIMCS_CUDA_ERROR;
    }
    *out = c;
    return 0;
}

int cimcs_nccl_unique_id(uint8_t* out, int32_t nbytes) {
    if (!out || nbytes < (int32_t)sizeof(ncclUniqueId))
        return fail(CIMCS_INPUT_ERROR, "need a 128-byte buffer");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return 0;
}

int cimcs_create_sharded(int32_t device, int32_t dtype, int32_t world, int32_t rank,
                         const uint8_t* nccl_id, cimcs_ctx** out) {
    if (world < 1 || rank < 0 || rank >= world || !nccl_id)
        return fail(CIMCS_CONFIG_ERROR, "bad world/rank/id");
    if (int rc = cimcs_create(device, dtype, out)) return rc;
    cimcs_ctx* c = *out;
    c->world = c->sh_world = world;
    c->rank = c->sh_rank = rank;
    c->sharded = c->sh_rows = true;
    if (world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        const ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            cimcs_destroy(c);
            *out = nullptr;
            return fail(CIMCS_CUDA_ERROR, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
    }
    return 0;
}

void cimcs_destroy(cimcs_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    free_problems(c);
    if (c->stage) cudaFree(c->stage);
    if (c->stage_i) cudaFree(c->stage_i);
    if (c->alt) cudaFree(c->alt);
    if (c->err) cudaFree(c->err);
    if (c->pump) cudaFree(c->pump);
    if (c->dTl) cudaFree(c->dTl);
    if (c->hist) cudaFree(c->hist);
    if (c->pin) cudaFreeHost(c->pin);
    if (c->pin_c0) cudaFreeHost(c->pin_c0);
    if (c->dc0) cudaFree(c->dc0);
    drop_graphs(c);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->side) cudaStreamDestroy(c->side);
    cudaStreamDestroy(c->stream);
    delete c;
}

int cimcs_set_option(cimcs_ctx* c, const char* key, int64_t v) {
    if (!c || !key) return fail(CIMCS_INPUT_ERROR, "null argument");
    const std::string k(key);
    if (k == "host_threads") c->host_threads = (int)std::max<int64_t>(1, v);
    else if (k == "use_graphs") c->use_graphs = v != 0;
    else if (k == "gram_tc") c->gram_tc = v > 0 ? 1 : (v < 0 ? -1 : 0);
    else if (k == "kernel_timing") {
        c->kernel_timing = v != 0;
        c->timing.tile_kernel_ms = 0.0;
        c->timing.tile_kernel_launches = 0;
        drop_graphs(c);
    } else if (k == "tile_shard") {
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set tile_shard before set_problems");
        c->tshard_opt = v != 0 ? 1 : 0;
    } else if (k == "mri_cluster") {
        c->mri_cluster = v != 0;
        drop_graphs(c);
    } else if (k == "gram_l2") {
        c->gram_l2 = v < 0 ? 0 : (int)v;
        drop_graphs(c);
    } else if (k == "pdl") {
        c->use_pdl = v != 0;
        drop_graphs(c);
    }
    else if (k == "timeline") {  // measurement aid: stamps of the last tile / update launch pair
        if (v != 0 && !c->dTl) {
            if (int rc = dalloc(c, &c->dTl, (size_t)kTlCap * 4 * 8)) return rc;
        } else if (v == 0 && c->dTl) {
            cudaStreamSynchronize(c->stream);
            cudaFree(c->dTl);
            c->dTl = nullptr;
        }
        drop_graphs(c);
    }
    else if (k == "sched_ctas") {  // measurement aid: persistent CTAs of the item schedules
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set sched_ctas before set_problems");
        c->sched_ctas = (int)std::max<int64_t>(0, v);
    }
    else if (k == "overlap_update") {
        c->overlap_upd = v != 0;
        drop_graphs(c);
    }
    else if (k == "cluster_loop") {
        c->use_cluster = v != 0;
        drop_graphs(c);
    }
    else if (k == "tensor_cores") {
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set tensor_cores before set_problems");
        c->want_tc = v != 0;
    } else if (k == "refit_compact") {
        c->cmp_opt = v != 0;
        drop_graphs(c);
    } else if (k == "sym64") {
        if (c->B > 0) return fail(CIMCS_CONFIG_ERROR, "set sym64 before set_problems");
        c->want_sym64 = v != 0;
    }
    else return fail(CIMCS_CONFIG_ERROR, "unknown option " + k);
    return 0;
}


int cimcs_get_timeline(cimcs_ctx* c, uint64_t* out, int64_t cap, int64_t* n) {
    if (!c || !out || !n) return fail(CIMCS_INPUT_ERROR, "null argument");
    if (!c->dTl) return fail(CIMCS_CONFIG_ERROR, "set option timeline = 1 first");
    *n = std::min<int64_t>(cap, (int64_t)kTlCap * 4);
    return copy_sync(c, out, c->dTl, (size_t)*n * 8, cudaMemcpyDeviceToHost);
}

}  // extern "C"
