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
    if (m < INT64_C(1792)) {
        if (m < INT64_C(159)) {
            if (n < INT64_C(1132)) {
                if (k < INT64_C(304)) {
                    if (k < INT64_C(144)) {
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
                if (m < INT64_C(12)) {
                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(28)) {
                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(405)) {
                            if (m < INT64_C(70)) {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(725)) {
                                    select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(444)) {
                if (m < INT64_C(1109)) {
                    if (n < INT64_C(111)) {
                        if (m < INT64_C(555)) {
                            select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(167)) {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(46)) {
                            select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(287)) {
                                if (m < INT64_C(555)) {
                                    if (n < INT64_C(203)) {
                                        if (m < INT64_C(278)) {
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
                                } else {
                                    if (n < INT64_C(144)) {
                                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(992)) {
                                            select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1537)) {
                                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(555)) {
                                    if (m < INT64_C(278)) {
                                        if (k < INT64_C(248)) {
                                            select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(46)) {
                        select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(167)) {
                            if (k < INT64_C(96)) {
                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(278)) {
                    if (n < INT64_C(544)) {
                        select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(405)) {
                            if (k < INT64_C(203)) {
                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(287)) {
                                    select_f32_nn_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(725)) {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(725)) {
                        if (n < INT64_C(992)) {
                            if (k < INT64_C(111)) {
                                if (m < INT64_C(784)) {
                                    select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(1145)) {
                                if (m < INT64_C(784)) {
                                    select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(1025)) {
                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(28)) {
            if (m < INT64_C(4435)) {
                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                return out;
            } else {
                if (m < INT64_C(35480)) {
                    select_f32_nn_config out = {4u, 2u, 8u, 64u, 1u};
                    return out;
                } else {
                    if (m < INT64_C(70960)) {
                        if (k < INT64_C(118)) {
                            select_f32_nn_config out = {4u, 2u, 8u, 64u, 1u};
                            return out;
                        } else {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(7168)) {
                if (n < INT64_C(363)) {
                    if (k < INT64_C(544)) {
                        if (n < INT64_C(46)) {
                            if (m < INT64_C(4435)) {
                                select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(314)) {
                                if (n < INT64_C(91)) {
                                    if (m < INT64_C(4435)) {
                                        select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 2u, 8u, 64u, 1u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(28)) {
                                        if (m < INT64_C(4435)) {
                                            select_f32_nn_config out = {4u, 2u, 8u, 64u, 1u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(444)) {
                                    select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        if (n < INT64_C(182)) {
                                            select_f32_nn_config out = {8u, 4u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(182)) {
                                if (k < INT64_C(815)) {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(91)) {
                        if (n < INT64_C(46)) {
                            if (k < INT64_C(63)) {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 2u, 8u, 64u, 1u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(97)) {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    }
                } else {
                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_F32_NN_H */
