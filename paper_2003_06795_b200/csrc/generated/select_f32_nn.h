#ifndef SELECT_F32_NN_H
#define SELECT_F32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nn_config;

static inline select_f32_nn_config select_f32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(448)) {
        if (m < INT64_C(12)) {
            select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
            return out;
        } else {
            if (n < INT64_C(144)) {
                if (n < INT64_C(79)) {
                    if (k < INT64_C(272)) {
                        select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                }
            } else {
                if (n < INT64_C(544)) {
                    if (m < INT64_C(139)) {
                        if (k < INT64_C(992)) {
                            if (n < INT64_C(227)) {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(70)) {
                                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(444)) {
                            if (k < INT64_C(992)) {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(1537)) {
                                        select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(70)) {
                        if (n < INT64_C(1132)) {
                            select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(405)) {
                                if (m < INT64_C(139)) {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(124)) {
                                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(405)) {
                                if (k < INT64_C(124)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(227)) {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(17740)) {
            if (n < INT64_C(444)) {
                if (m < INT64_C(4435)) {
                    if (n < INT64_C(176)) {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(222)) {
                                if (k < INT64_C(167)) {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(46)) {
                                if (m < INT64_C(2218)) {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(28)) {
                                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(2218)) {
                                    if (k < INT64_C(444)) {
                                        if (k < INT64_C(314)) {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(46)) {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(1537)) {
                                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(168)) {
                        if (n < INT64_C(222)) {
                            if (n < INT64_C(28)) {
                                if (m < INT64_C(8870)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(56)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(118)) {
                                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(182)) {
                            if (m < INT64_C(8870)) {
                                if (n < INT64_C(91)) {
                                    if (k < INT64_C(222)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(91)) {
                                    if (k < INT64_C(222)) {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(1792)) {
                    if (k < INT64_C(111)) {
                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(1449)) {
                            if (n < INT64_C(992)) {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(405)) {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(1109)) {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                }
            }
        } else {
            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
            return out;
        }
    }
}

#endif /* SELECT_F32_NN_H */
